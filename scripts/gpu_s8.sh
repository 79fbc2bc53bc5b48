#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s8; mkdir -p $O
timeout 1200 python scripts/ab_time.py --libs ab/v3.so,ab/head_prev.so,ab/new.so --configs c2,c3,c5 --rounds 2 > $O/ab_ticket.jsonl 2> $O/ab.err
for l in v3 head_prev new; do SPCONV_LIB=$PWD/ab/$l.so timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2_$l.json 2>> $O/ab.err; done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pipe_kernel --launch-skip 3 --launch-count 30 --csv --log-file $O/launches_c2_timed.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 0 --launch-count 66 --csv --log-file $O/launches_c2_all.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $O/ncu_launches2.log 2>&1
echo done >> $O/summary.txt
