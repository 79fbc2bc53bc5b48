#!/bin/bash
# NEXT-2/3 blocks: R = 4 vs R = 2 (more units when a layer has fewer units than SMs)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s41; mkdir -p $O
timeout 600 python scripts/blocks_bench.py > $O/blocks_default.jsonl 2> $O/err1
SPCONV_PIPE_R=2 timeout 600 python scripts/blocks_bench.py > $O/blocks_r2.jsonl 2> $O/err2
timeout 900 python scripts/ab_time.py --configs "custom:256,32,16,16,32,0.2;custom:16,512,28,28,512,0.058;custom:16,512,28,28,512,0.01;custom:16,256,28,28,512,0.242" --kernels pipe,generic --rounds 1 --envs ";SPCONV_PIPE_R=2" > $O/layers.jsonl 2> $O/err3
echo done >> $O/summary.txt
