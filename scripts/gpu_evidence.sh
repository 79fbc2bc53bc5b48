#!/bin/bash
# Round evidence pass on one B200: GPU tests, smoke, the default bench line (c2),
# bench lines for every config, the reference arm, the ncu launch list of the
# default bench command and one `ncu --set full` capture per headline config.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
: > gpurun_out/bench_all.jsonl
for c in c1 c2 c3 c4_50 c4_80 c4_90 c4_95 c5; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
   --log-file gpurun_out/launches_c2.csv python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for c in c2 c3 c4_50 c4_80 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pipe_kernel -s 3 -c 1 \
     -o gpurun_out/full_$c -f python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/full_$c.log 2>&1
  # summarise on the box (the reports together exceed gpurun's 64 MiB copy-back); keep c2's report
  fl=$(python -c "import synthgen; print(synthgen.CONFIGS['$c'].useful_flops)")
  la=""; [ "$c" = c2 ] && la="--launches gpurun_out/launches_c2.csv"
  python scripts/ncu_summary.py gpurun_out/full_$c.ncu-rep gpurun_out/r01_${c}_pipe_full --config $c --flops $fl $la \
     --traffic-json gpurun_out/ncu_traffic.json > /dev/null 2>> gpurun_out/ncu_summary.err
  [ "$c" = c2 ] || rm -f gpurun_out/full_$c.ncu-rep
done
timeout 600 python scripts/breakeven.py --shape c2 > gpurun_out/breakeven_c2.jsonl 2> gpurun_out/breakeven_c2.err
timeout 600 python scripts/breakeven.py --shape c4 > gpurun_out/breakeven_c4.jsonl 2> gpurun_out/breakeven_c4.err
timeout 600 python scripts/lstm_bench.py --batch 64 --reps 10 > gpurun_out/lstm_b64.jsonl 2>&1
timeout 600 python scripts/lstm_bench.py --batch 1 --reps 10 > gpurun_out/lstm_b1.jsonl 2>&1
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
echo done
