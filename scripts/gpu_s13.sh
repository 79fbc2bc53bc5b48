#!/bin/bash
# final evidence of round 2: full suite, smoke, benches of every config, c4 break-even,
# ncu --set full for c4 (7-row tiles) summarised on the box
cd $GRAFT_REPO_ROOT
O=gpurun_out/s13; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
for c in c1 c2 c3 c4_50 c4_80 c4_90 c4_95 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c exit $?" >> $O/summary.txt
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default exit $?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench reference exit $?" >> $O/summary.txt
timeout 1200 python scripts/breakeven.py --shape c4 > $O/breakeven_c4.jsonl 2> $O/breakeven_c4.err
flops() { python -c "import synthgen; print(synthgen.CONFIGS['$1'].useful_flops)"; }
for c in c4_95 c4_80 c4_50; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 3 -c 1 -o $O/full_$c -f python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > $O/full_$c.log 2>&1
  python scripts/ncu_summary.py $O/full_$c.ncu-rep $O/r02_${c}_t7_full --config $c --flops $(flops $c) > /dev/null 2>> $O/summ.err
done
rm -f $O/*.ncu-rep
echo done >> $O/summary.txt
