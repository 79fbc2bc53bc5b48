#!/bin/bash
# after the sk_split refactor (plan-free core + test-only ABI): GPU suite subset + timing sanity
cd $GRAFT_REPO_ROOT
O=gpurun_out/s53; mkdir -p $O
timeout 900 python -m pytest tests -q -p no:cacheprovider -k "split or stress or stream_k or abi or bench_configuration" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --configs c2,c3,c4_50 --rounds 1 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
