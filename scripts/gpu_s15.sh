#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s15; mkdir -p $O
timeout 600 python scripts/host_overhead.py ab/preramp.so,ab/cache.so > $O/host_overhead.jsonl 2> $O/ho.err
timeout 600 python scripts/e2e_ab.py ab/preramp.so,ab/cache.so > $O/e2e.jsonl 2> $O/e2e.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "forward_host or concurrent or stream_k or graph or very_wide or batch_zero or unaligned" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
