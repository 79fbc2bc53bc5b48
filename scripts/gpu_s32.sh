#!/bin/bash
# bound on the epilogue stores: the same build with the output stores predicated off
cd $GRAFT_REPO_ROOT
O=gpurun_out/s32; mkdir -p $O
timeout 1200 python scripts/ab_time.py --libs ab/head.so,ab/nostore.so --configs c2,c3 --rounds 2 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
