#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s17; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
SPCONV_DEBUG=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/pytest_debug.log 2>&1; echo "pytest debug exit $?" >> $O/summary.txt
SPCONV_PDL=0 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "stream_k or bench_configuration or dense or graph" > $O/pytest_nopdl.log 2>&1; echo "pytest nopdl exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --configs c5 --densities 1.0 --kernel dense --rounds 1 > $O/dense_c5.jsonl 2>&1
echo done >> $O/summary.txt
