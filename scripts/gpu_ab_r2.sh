#!/bin/bash
# A/B of the pipe kernel's rows per group (R = 4 default vs R = 2 with 11-12 warps):
# GPU parity suite under SPCONV_PIPE_R=2, then bench lines for both on every config.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
SPCONV_PIPE_R=2 timeout 900 python -m pytest tests -m gpu -q -k "not lstm" > gpurun_out/pytest_r2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2.log
: > gpurun_out/ab_r2.jsonl
for c in ${BENCH_CONFIGS:-c2 c3 c4_50 c4_80 c4_90 c4_95 c5}; do
  for r in 4 2 4 2; do
    timeout 300 python bench.py --config $c --rows $r --steps ${STEPS:-300} --warmup 5 --no-cpu-baseline \
      | sed "s/^/R$r $c /" >> gpurun_out/ab_r2.jsonl 2>> gpurun_out/ab_r2.err
  done
done
echo done
