#!/bin/bash
# ncu --set full summaries of the final build for c5, c4_50, c4_95 and the dense kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/s56; mkdir -p $O
flops() { python -c "import synthgen; c=synthgen.CONFIGS['$1']; c=c.with_density($2) if $2 else c; print(c.useful_flops)"; }
for c in c5 c4_50 c4_95; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 3 -c 1 -o $O/full_$c -f python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > $O/full_$c.log 2>&1
  python scripts/ncu_summary.py $O/full_$c.ncu-rep $O/r02_${c}_final_full --config $c --flops $(flops $c 0) > /dev/null 2>> $O/summ.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 3 -c 1 -o $O/full_dense_c2 -f python scripts/ab_time.py --child c2 1.0 --kernel dense --iters 3 --reps 1 > $O/full_dense_c2.log 2>&1
python scripts/ncu_summary.py $O/full_dense_c2.ncu-rep $O/r02_dense_c2_d1_final_full --config c2@1.0 --flops $(flops c2 1.0) > /dev/null 2>> $O/summ.err
rm -f $O/*.ncu-rep
echo done >> $O/summary.txt
