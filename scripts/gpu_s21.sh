#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s21; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "wide or edge or random or stream_k or seven or fused or launch_info or auto" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/cache.so,ab/wide2.so --configs c2,c3,c5,c4_80 --rounds 2 > $O/ab_wide.jsonl 2> $O/ab.err
timeout 900 python scripts/ab_time.py --libs ab/cache.so,ab/wide2.so --configs "custom:8,64,224,224,64,0.2;custom:16,128,112,112,128,0.2" --rounds 1 --iters 10 >> $O/ab_wide.jsonl 2>> $O/ab.err
echo done >> $O/summary.txt
