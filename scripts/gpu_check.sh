#!/bin/bash
# One gpurun pass: GPU parity tests, smoke, bench on every config, ncu launch list and
# one --set full capture of the top kernel on c2.  Writes everything under gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
: > gpurun_out/bench.jsonl
for c in ${BENCH_CONFIGS:-c2 c3 c4_50 c4_80 c4_90 c4_95 c5}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-200} --warmup 5 ${BENCH_EXTRA:-} >> gpurun_out/bench.jsonl 2>> gpurun_out/bench.err
done
if [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled -s 3 -c 1 \
     -o gpurun_out/prof_c2 -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
fi
echo done
