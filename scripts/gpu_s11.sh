#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s12; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "seven or c4 or random or edge or graph or debug" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
timeout 1200 python scripts/ab_time.py --libs ab/lanemap.so,ab/t7b.so --configs c4_50,c4_80,c4_90,c4_95 --rounds 2 > $O/ab_t7.jsonl 2> $O/ab.err
timeout 900 python scripts/ab_time.py --libs ab/lanemap.so,ab/t7b.so --configs "custom:16,512,28,28,512,0.01;custom:16,512,28,28,512,0.058;custom:16,256,28,28,512,0.242" --rounds 1 --iters 20 >> $O/ab_t7.jsonl 2>> $O/ab.err

timeout 900 python scripts/blocks_bench.py > gpurun_out/s12/blocks.jsonl 2> gpurun_out/s12/blocks.err
echo done >> gpurun_out/s12/summary.txt
