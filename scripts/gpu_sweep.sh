#!/bin/bash
# Bench sweep: configs x rows-per-group variants (kernel-only, no CPU baseline).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3 c5}; do
  for r in ${ROWS:-4 8}; do
    timeout 300 python bench.py --config $c --rows $r --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline ${EXTRA:-} >> gpurun_out/sweep.jsonl 2>>gpurun_out/sweep.err
  done
done
