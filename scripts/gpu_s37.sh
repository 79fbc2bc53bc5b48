#!/bin/bash
# per-warp split clamped to one stage around the CTA-level split: c4_50 regression check
cd $GRAFT_REPO_ROOT
O=gpurun_out/s37; mkdir -p $O
timeout 1500 python scripts/ab_time.py --libs ab/wide2.so,ab/head.so,ab/clamp.so --configs "c4_50;c2;c3;custom:40,48,40,40,40,0.2" --rounds 2 > $O/ab.jsonl 2> $O/ab.err
timeout 600 python scripts/ab_time.py --libs ab/clamp.so --configs "c4_50;c2;c3" --rounds 1 --envs "SPCONV_PIPE_SK_SPLIT=uniform" >> $O/ab.jsonl 2>> $O/ab.err
echo done >> $O/summary.txt
