#!/bin/bash
# fused epilogue: straight-line pooling (predicated stores, one 64-bit base per pooled row)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s44; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fused or bench_configuration_c3 or random or edge or stress" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --libs ab/head.so,ab/fepi.so --configs c3,c2 --rounds 3 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
