#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s14; mkdir -p $O
timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_driver.json 2> $O/bench_driver.err; echo "bench exit $?" >> $O/summary.txt
timeout 600 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?" >> $O/summary.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 600 python scripts/e2e_ab.py > $O/e2e.jsonl 2> $O/e2e.err
echo done >> $O/summary.txt
