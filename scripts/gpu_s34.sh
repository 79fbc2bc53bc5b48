#!/bin/bash
# c4: 128 units on 148 SMs at 8 warps per CTA; 7 or 6 warps -> more (ragged) group sets, stream-K
cd $GRAFT_REPO_ROOT
O=gpurun_out/s34; mkdir -p $O
timeout 1500 python scripts/ab_time.py --libs ab/head.so --configs c4_80,c4_90,c4_95,c2 --rounds 2 --envs ";SPCONV_PIPE_GPC=7;SPCONV_PIPE_GPC=6" > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
