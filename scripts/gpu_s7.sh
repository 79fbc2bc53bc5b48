#!/bin/bash
# GPU session 7: full suite, benches, ncu evidence (launch list + --set full captures,
# summarised ON THE BOX; the .ncu-rep files are deleted: gpurun copies back <= 64 MiB)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s7; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
for c in c2 c3 c5 c4_50 c4_80 c4_90 c4_95 c1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c exit $?" >> $O/summary.txt
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default exit $?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
flops() { python -c "import synthgen; c=synthgen.CONFIGS['$1']; c=c.with_density($2) if $2 else c; print(c.useful_flops)"; }
for spec in "c2 pipe_kernel 0" "c3 pipe_kernel 0" "c4_95 pipe_kernel 0" "c5 pipe_kernel 0"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $O/full_$1 -f python bench.py --config $1 --steps 30 --warmup 3 --no-cpu-baseline > $O/full_$1.log 2>&1
  python scripts/ncu_summary.py $O/full_$1.ncu-rep $O/r02_$1_full --config $1 --flops $(flops $1 0) > /dev/null 2>> $O/summ.err
done
python scripts/ncu_summary.py $O/full_c2.ncu-rep $O/r02_c2_full_launches --config c2 --flops $(flops c2 0) --launches $O/launches_c2.csv > /dev/null 2>> $O/summ.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 3 -c 1 -o $O/full_dense_c2 -f python scripts/ab_time.py --child c2 1.0 --kernel dense --iters 3 --reps 1 > $O/full_dense_c2.log 2>&1
python scripts/ncu_summary.py $O/full_dense_c2.ncu-rep $O/r02_dense_c2_d1_full --config c2@1.0 --flops $(flops c2 1.0) > /dev/null 2>> $O/summ.err
ls -la $O > $O/listing.txt
rm -f $O/*.ncu-rep
echo done >> $O/summary.txt
