#!/bin/bash
# final validation of HEAD: full GPU suite (incl. the 48-layer stream-K stress), smoke,
# bench default (c2) and c3
cd $GRAFT_REPO_ROOT
O=gpurun_out/s45; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default exit $?" >> $O/summary.txt
timeout 900 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 exit $?" >> $O/summary.txt
echo done >> $O/summary.txt
