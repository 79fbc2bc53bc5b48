#!/bin/bash
# per-CTA end-time spread: work content (bid) or SM?  Same c2/c3 launches with the
# work index reversed (SPCONV_PIPE_REV=1: CTA with ticket t does the work of G-1-t)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s24; mkdir -p $O
SPCONV_PIPE_TRACE=$O/trace_c2.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_REV=1 SPCONV_PIPE_TRACE=$O/trace_c2_rev.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c3.txt timeout 300 python scripts/ab_time.py --configs c3 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_REV=1 SPCONV_PIPE_TRACE=$O/trace_c3_rev.txt timeout 300 python scripts/ab_time.py --configs c3 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
echo done >> $O/summary.txt
