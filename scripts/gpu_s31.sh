#!/bin/bash
# per-warp stream-K split (default): full GPU suite + debug-mode stream-K tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/s31; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
SPCONV_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "stream_k or split or bench_configuration" > $O/pytest_debug.log 2>&1; echo "pytest debug exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
