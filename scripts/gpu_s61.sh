#!/bin/bash
# per-call R = 2 alternate plan: full GPU suite + A/B against SPCONV_NO_ALT=1
cd $GRAFT_REPO_ROOT
O=gpurun_out/s61; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1500 python scripts/ab_time.py --configs c4_80,c2,c3,c5,c4_90 --rounds 2 --envs ";SPCONV_NO_ALT=1" > $O/ab.jsonl 2> $O/ab.err
timeout 1200 python scripts/ab_time.py --configs c2,c4_80,c5 --batches 2,4,8,16,24 --rounds 1 --envs ";SPCONV_NO_ALT=1" > $O/ab_batches.jsonl 2>> $O/ab.err
timeout 600 python scripts/blocks_bench.py > $O/blocks.jsonl 2> $O/blocks.err
SPCONV_NO_ALT=1 timeout 600 python scripts/blocks_bench.py > $O/blocks_noalt.jsonl 2>> $O/blocks.err
echo done >> $O/summary.txt
