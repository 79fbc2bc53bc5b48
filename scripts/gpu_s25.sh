#!/bin/bash
# realigned 16-byte stores in the shifted (XS = 3) conv epilogue: parity + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s25; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "bench_configuration or random or edge or epilogue or block or wide or stream_k or staging" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/cache.so,ab/vec.so --configs c2,c5,c3,c4_80 --rounds 2 > $O/ab_vec.jsonl 2> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c2.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
echo done >> $O/summary.txt
