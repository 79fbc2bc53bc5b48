#!/bin/bash
# generic kernel with 8 independent tap loads per step: parity + small-call timings (old vs new)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s39; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "generic or random or edge or small or epilogue or block or resize" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1500 python scripts/ab_time.py --libs ab/head.so,ab/gen.so --configs c1,c2,c4_95,c3 --batches 1,2,4,8,16 --kernels generic,pipe --rounds 1 --iters 50 > $O/small.jsonl 2> $O/ab.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
echo done >> $O/summary.txt
