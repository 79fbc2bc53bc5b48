#!/bin/bash
# sk_split with O(1) lane prefix costs: split / stress tests + timing sanity
cd $GRAFT_REPO_ROOT
O=gpurun_out/s43; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "split or stress or stream_k" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --libs ab/head.so --configs c2,c3,c4_50 --rounds 1 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
