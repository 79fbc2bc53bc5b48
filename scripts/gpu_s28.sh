#!/bin/bash
# per-warp cost-balanced stream-K split points: parity (stream-K tests) + A/B + trace
cd $GRAFT_REPO_ROOT
O=gpurun_out/s28; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or bench_configuration or skipped or graph or concurrent" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/cache.so,ab/split.so,ab/split2.so --configs c2,c3,c5 --rounds 2 > $O/ab_split.jsonl 2> $O/ab.err
timeout 600 python scripts/ab_time.py --libs ab/split2.so --configs c2,c3 --rounds 1 --envs "SPCONV_PIPE_SK_SPLIT=uniform" >> $O/ab_split.jsonl 2>> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c2.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c3.txt timeout 300 python scripts/ab_time.py --configs c3 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
echo done >> $O/summary.txt
