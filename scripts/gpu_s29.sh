#!/bin/bash
# split2 per-CTA trend: work index or arrival order?  (REV maps work index G-1-t to ticket t)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s29; mkdir -p $O
SPCONV_PIPE_TRACE=$O/trace_c2.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_REV=1 SPCONV_PIPE_TRACE=$O/trace_c2_rev.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_SK_SPLIT=uniform SPCONV_PIPE_TRACE=$O/trace_c2_uni.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
echo done >> $O/summary.txt
