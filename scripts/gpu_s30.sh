#!/bin/bash
# c5 (no stream-K) +1% with the split build: kernel-parameter size or the empty-range branch?
cd $GRAFT_REPO_ROOT
O=gpurun_out/s30; mkdir -p $O
timeout 1500 python scripts/ab_time.py --libs ab/cache.so,ab/wide2.so,ab/split2.so,ab/tab1.so,ab/noskip.so --configs c5,c2 --rounds 2 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
