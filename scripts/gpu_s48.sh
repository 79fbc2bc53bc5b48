#!/bin/bash
# stage size re-check on the final build (per-warp split): 80 KB (2 stages) vs ~56-60 KB (3 stages)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s48; mkdir -p $O
timeout 1500 python scripts/ab_time.py --libs ab/head.so --configs "c4_50;c4_80;c4_95;c5;custom:8,64,224,224,64,0.2;custom:16,256,28,28,512,0.242" --rounds 2 --envs ";SPCONV_PIPE_STAGE_BYTES=90112;SPCONV_PIPE_STAGE_BYTES=98304" > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
