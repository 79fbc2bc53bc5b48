#!/bin/bash
# split cost over active lanes: ragged group sets (F = 40) split test + c2/c3 timing
cd $GRAFT_REPO_ROOT
O=gpurun_out/s35; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "split or stream_k" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --libs ab/head.so --configs "c2;c3;custom:40,48,40,40,40,0.2" --rounds 1 --envs ";SPCONV_PIPE_SK_SPLIT=uniform" > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
