#!/bin/bash
# full GPU suite + smoke + default bench on the committed build; c3 fused vs the same
# layer conv-only; c2/c3 per-CTA trace (start, head parked, end, tail wait)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s22; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench.err; echo "bench exit $?" >> $O/summary.txt
timeout 900 python scripts/ab_time.py --configs "c3;custom:32,64,56,56,64,0.1" --rounds 2 > $O/c3_vs_conv.jsonl 2>> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c2.txt timeout 300 python scripts/ab_time.py --configs c2 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
SPCONV_PIPE_TRACE=$O/trace_c3.txt timeout 300 python scripts/ab_time.py --configs c3 --rounds 1 --iters 3 > /dev/null 2>> $O/ab.err
echo done >> $O/summary.txt
