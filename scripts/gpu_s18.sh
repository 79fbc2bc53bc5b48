#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s18; mkdir -p $O
for r in 1 2; do for c in c2 c3 c4_95; do for l in cache prologue; do
  SPCONV_LIB=$PWD/ab/$l.so timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline 2>>$O/err.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['timing']
print(json.dumps({'lib':'$l','config':'$c','median_us':t['median_ms']*1e3,'warm_us':t['warm_l2_median_ms']*1e3,'steady_us':t['steady_state_ms']*1e3}))" >> $O/ab_prologue.jsonl
done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or dense or bench_configuration or graph or seven" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
SPCONV_DEBUG=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/pytest_debug.log 2>&1; echo "pytest debug exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
