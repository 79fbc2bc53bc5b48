#!/bin/bash
# bench protocol numbers (flushed / warm / steady) for the split build vs the previous commit's
cd $GRAFT_REPO_ROOT
O=gpurun_out/s33; mkdir -p $O
for i in 1 2; do
cp ab/head.so paper_2005_04091_b200/libspconv.so
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench_head_$i.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 > $O/bench_head_c3_$i.json 2>> $O/bench.err
cp ab/wide2.so paper_2005_04091_b200/libspconv.so
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench_prev_$i.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 50 --warmup 5 > $O/bench_prev_c3_$i.json 2>> $O/bench.err
done
cp ab/head.so paper_2005_04091_b200/libspconv.so
echo done >> $O/summary.txt
