#!/bin/bash
# random stream-K stress (per-warp split, R = 2 / 4, column blocks, 7/8-row tiles)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s42; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stress" --durations=3 > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
