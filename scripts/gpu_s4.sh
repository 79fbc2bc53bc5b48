#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "dense or very_wide or auto or stream_k or bench_configuration" > $O/pytest_dense.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --configs c2,c4_50,c5 --densities 1.0 --kernel dense --rounds 1 > $O/dense.jsonl 2> $O/dense.err
timeout 1200 python scripts/breakeven.py --shape c2 > $O/breakeven_c2.jsonl 2> $O/breakeven_c2.err
timeout 1200 python scripts/breakeven.py --shape c4 > $O/breakeven_c4.jsonl 2> $O/breakeven_c4.err
timeout 1200 python scripts/breakeven.py --shape c5 --n 32 > $O/breakeven_c5.jsonl 2> $O/breakeven_c5.err
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
