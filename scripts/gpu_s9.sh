#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s9; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "c4 or c1 or edge or random or two_rows or debug or staging" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/new.so,ab/lane.so --configs c4_50,c4_80,c4_90,c4_95,c2 --rounds 2 > $O/ab_lane.jsonl 2> $O/ab.err
timeout 600 ncu --set full --clock-control none -k regex:pipe_kernel -s 3 -c 1 -o $O/full_c4_95 -f python bench.py --config c4_95 --steps 30 --warmup 3 --no-cpu-baseline > $O/full_c4_95.log 2>&1
python scripts/ncu_summary.py $O/full_c4_95.ncu-rep $O/r02_c4_95_lane_full --config c4_95 --flops $(python -c "import synthgen; print(synthgen.CONFIGS['c4_95'].useful_flops)") > /dev/null 2>> $O/summ.err
rm -f $O/*.ncu-rep
echo done >> $O/summary.txt
