#!/bin/bash
# phase clock sums (-DSPC_PROF build): epilogue split into park / resume / end barrier / prologue
cd $GRAFT_REPO_ROOT
O=gpurun_out/s26; mkdir -p $O
for c in c2 c3 c5 c4_95; do
SPCONV_PIPE_PROF=$O/prof_$c.txt timeout 300 python scripts/ab_time.py --libs ab/prof.so --configs $c --rounds 1 --iters 5 > $O/t_$c.jsonl 2>> $O/ab.err
done
echo done >> $O/summary.txt
