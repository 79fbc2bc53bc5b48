#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s16; mkdir -p $O
timeout 1200 python scripts/ab_time.py --configs c2,c5 --densities 1.0 --kernel dense --envs "SPCONV_DENSE_STAGE_BYTES=20480;SPCONV_DENSE_STAGE_BYTES=40960;SPCONV_DENSE_STAGE_BYTES=61440;SPCONV_DENSE_STAGE_BYTES=81920" --rounds 2 > $O/dense_stage.jsonl 2> $O/ab.err
timeout 900 python scripts/ab_time.py --configs c4_50 --envs "SPCONV_PIPE_R=2;SPCONV_PIPE_R=4" --rounds 2 >> $O/r_ab.jsonl 2>> $O/ab.err
timeout 900 python scripts/ab_time.py --configs c2 --densities 0.3,0.4,0.5 --envs "SPCONV_PIPE_R=2;SPCONV_PIPE_R=4" --kernel pipe --rounds 1 >> $O/r_ab.jsonl 2>> $O/ab.err
echo done >> $O/summary.txt
