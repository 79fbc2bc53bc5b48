#!/bin/bash
# GPU session 1 (round 2): correctness of dispatcher variants, A/B timing, phase profile, baseline bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/gpu.txt
for v in 1 2 3 4 5; do
  SPCONV_LIB=$PWD/ab/v$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c2 or c3 or stream_k or random_shapes" > gpurun_out/s1/pytest_v$v.log 2>&1
  echo "v$v exit $?" >> gpurun_out/s1/pytest_summary.txt
done
timeout 900 python scripts/ab_time.py --libs ab/v0.so,ab/v1.so,ab/v2.so,ab/v3.so,ab/v4.so,ab/v5.so --configs c2,c3,c5,c4_80 --rounds 2 > gpurun_out/s1/ab_variants.jsonl 2> gpurun_out/s1/ab_variants.err
SPCONV_PIPE_PROF=$PWD/gpurun_out/s1/prof_c2.txt timeout 300 python scripts/ab_time.py --libs ab/prof_v0.so --configs c2,c3 --rounds 1 --iters 5 --reps 2 > gpurun_out/s1/prof_ab.jsonl 2>&1
timeout 900 python scripts/ab_time.py --libs ab/v0.so --configs c2 --densities 0.01,0.02,0.05,0.1,0.2,0.3 --rounds 1 > gpurun_out/s1/dens_v0.jsonl 2>&1
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/s1/bench_c2.json 2> gpurun_out/s1/bench_c2.err
echo done
