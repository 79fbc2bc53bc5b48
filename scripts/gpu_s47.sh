#!/bin/bash
# stage size re-check on the final build (per-warp split): 80 KB (2 stages) vs ~56-60 KB (3 stages)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s47; mkdir -p $O
timeout 1500 python scripts/ab_time.py --libs ab/head.so --configs c2,c3,c5 --rounds 2 --envs ";SPCONV_PIPE_STAGE_BYTES=98304;SPCONV_PIPE_STAGE_BYTES=110592" > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
