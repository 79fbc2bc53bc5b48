#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "dense or very_wide or auto" > $O/pytest_dense.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --configs c2 --densities 0.2,0.5,1.0 --kernel dense --rounds 1 > $O/dense_c2.jsonl 2> $O/dense_c2.err
timeout 900 python scripts/ab_time.py --configs c4_50,c5 --densities 1.0 --kernel dense --rounds 1 >> $O/dense_c2.jsonl 2>> $O/dense_c2.err
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench exit $?" >> $O/summary.txt
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
echo done >> $O/summary.txt
