#!/bin/bash
# GPU session 2: full GPU suite on the round-2 code, smoke, bench (new protocol), FFMA probe, sanitizers
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench exit $?" >> $O/summary.txt
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 ./scripts/probes/ffma_probe > $O/ffma_probe.log 2>&1
for tool in memcheck synccheck racecheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > $O/sanitize_$tool.log 2>&1
  echo "sanitize $tool exit $?" >> $O/summary.txt
done
echo done >> $O/summary.txt
