#!/bin/bash
# per-call R = 2 alternate with the stream-K overhead term: batch sweep A/B + the alt tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/s62; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "alternate or auto or bench_configuration or graph" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1500 python scripts/ab_time.py --configs c2,c4_80,c3 --batches 8,12,16,20,24,32,64 --rounds 1 --envs ";SPCONV_NO_ALT=1" > $O/ab_batches.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
