#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s10; mkdir -p $O
timeout 1200 python scripts/ab_time.py --libs ab/new.so,ab/lane.so,ab/lanemap.so --configs c2,c3,c5,c4_80,c4_95 --rounds 2 > $O/ab_lanemap.jsonl 2> $O/ab.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
