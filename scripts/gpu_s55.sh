#!/bin/bash
# stability: the full GPU suite three times back to back, then the parity suite with
# SPCONV_DEBUG=1 (stream self-check at create, a synchronised check of every call) and
# with programmatic dependent launch off
cd $GRAFT_REPO_ROOT
O=gpurun_out/s55; mkdir -p $O
for i in 1 2 3; do
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$i.log 2>&1; echo "pytest run $i exit $?" >> $O/summary.txt
done
SPCONV_DEBUG=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/pytest_debug.log 2>&1; echo "pytest debug exit $?" >> $O/summary.txt
SPCONV_PDL=0 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/pytest_nopdl.log 2>&1; echo "pytest nopdl exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
