#!/bin/bash
# round-2 final evidence (per-warp stream-K split build): full suite, smoke, benches of
# every config + reference arm, c2 launch list, ncu --set full of c2 / c3 summarised on
# the box, phase clocks (-DSPC_PROF build)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s38; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
for c in c2 c3 c5 c4_50 c4_80 c4_90 c4_95 c1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c exit $?" >> $O/summary.txt
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default exit $?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench reference exit $?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
flops() { python -c "import synthgen; print(synthgen.CONFIGS['$1'].useful_flops)"; }
for c in c2 c3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 3 -c 1 -o $O/full_$c -f python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > $O/full_$c.log 2>&1
  python scripts/ncu_summary.py $O/full_$c.ncu-rep $O/r02_${c}_split_full --config $c --flops $(flops $c) > /dev/null 2>> $O/summ.err
done
python scripts/ncu_summary.py $O/full_c2.ncu-rep $O/r02_c2_split_full_launches --config c2 --flops $(flops c2) --launches $O/launches_c2.csv > /dev/null 2>> $O/summ.err
for c in c2 c3; do
  SPCONV_PIPE_PROF=$O/phase_$c.txt timeout 300 python scripts/ab_time.py --libs ab/prof.so --configs $c --rounds 1 --iters 5 > /dev/null 2>> $O/ab.err
done
rm -f $O/*.ncu-rep
echo done >> $O/summary.txt
