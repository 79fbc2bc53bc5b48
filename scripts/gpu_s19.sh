#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s19; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or bench_configuration or skipped or mask or two_rows or seven or dense" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/cache.so,ab/costsk.so --configs c2,c3,c4_50 --rounds 3 > $O/ab_costsk.jsonl 2> $O/ab.err
for r in 1 2; do for c in c2 c3; do for l in cache costsk; do
  SPCONV_LIB=$PWD/ab/$l.so timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline 2>>$O/err.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['timing']
print(json.dumps({'lib':'$l','config':'$c','median_us':t['median_ms']*1e3,'warm_us':t['warm_l2_median_ms']*1e3,'steady_us':t['steady_state_ms']*1e3}))" >> $O/bench_costsk.jsonl
done; done; done
echo done >> $O/summary.txt
