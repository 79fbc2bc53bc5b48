#!/bin/bash
# final evidence after the stage-target change: full suite, smoke, benches of every
# config, the default bench line and the reference arm
cd $GRAFT_REPO_ROOT
O=gpurun_out/s64; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
for c in c2 c3 c5 c4_50 c4_80 c4_90 c4_95 c1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c exit $?" >> $O/summary.txt
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default exit $?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench reference exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
