#!/bin/bash
# small layers: kernel choice data for the AUTO cost model (verdict r1 item 6)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s6; mkdir -p $O
timeout 900 python scripts/ab_time.py --configs c1 --batches 1,2,4,8,16 --kernels pipe,tiled,generic --rounds 1 --iters 50 > $O/small_c1.jsonl 2> $O/small.err
timeout 900 python scripts/ab_time.py --configs c4_95 --batches 1,2,4,8,16,64 --kernels pipe,tiled,generic --rounds 1 --iters 20 > $O/small_c4.jsonl 2>> $O/small.err
timeout 900 python scripts/ab_time.py --configs c2 --batches 1,2,4 --kernels pipe,tiled,generic --rounds 1 --iters 20 > $O/small_c2.jsonl 2>> $O/small.err
timeout 900 python scripts/ab_time.py --configs "custom:16,512,28,28,512,0.01;custom:16,512,28,28,512,0.058;custom:16,256,28,28,512,0.242" --kernels pipe,tiled,generic --rounds 1 --iters 10 > $O/vgg.jsonl 2>> $O/small.err
timeout 900 python scripts/ab_time.py --configs c2 --envs "SPCONV_PIPE_STAGE_BYTES=20480;SPCONV_PIPE_STAGE_BYTES=40960;SPCONV_PIPE_STAGE_BYTES=81920" --rounds 2 > $O/stage_bytes.jsonl 2>> $O/small.err
echo done > $O/summary.txt
