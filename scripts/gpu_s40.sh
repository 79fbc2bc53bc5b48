#!/bin/bash
# dispatcher variant 6 (reload fused into the first tap of a channel): parity + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/s40; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or split or bench_configuration or random or edge or skipped or seven or wide or staging" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
SPCONV_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or split or random or skipped" > $O/pytest_debug.log 2>&1; echo "pytest debug exit $?" >> $O/summary.txt
timeout 1500 python scripts/ab_time.py --libs ab/head.so,ab/fr.so --configs c2,c3,c5,c4_50,c4_80,c4_95 --rounds 2 > $O/ab.jsonl 2> $O/ab.err
echo done >> $O/summary.txt
