#!/bin/bash
# ncu --set full capture of one launch of the hot kernel for a config (1 GPU).
# usage: bash scripts/gpu_prof.sh <config> <kernel-regex> <out-name> [bench args...]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cfg=$1; rx=$2; out=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 \
   -o gpurun_out/$out -f python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/$out.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$out.log
