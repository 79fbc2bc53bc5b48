#!/bin/bash
# L2 prefetch of the first stage at kernel start: bench protocol (flushed / warm / steady)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s52; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "stream_k or bench_configuration or seven or wide or staging or stress" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
for i in 1 2; do
for lib in head pf; do
  cp ab/$lib.so paper_2005_04091_b200/libspconv.so
  for c in c2 c3 c4_80; do
    timeout 600 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline > $O/b_${lib}_${c}_$i.json 2>> $O/err
  done
done
cp ab/pf.so paper_2005_04091_b200/libspconv.so
for c in c2 c3; do SPCONV_PIPE_PREFETCH=0 timeout 600 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline > $O/b_pfoff_${c}_$i.json 2>> $O/err; done
done
echo done >> $O/summary.txt
