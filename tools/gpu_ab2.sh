#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ab2.txt
for v in 1 0 1 0; do for c in c1 c2; do
  BM_CARVEOUT=$v BM_TIMELINE=1 timeout 300 python tools/chunk_prof.py $c 60 > gpurun_out/ab2_${c}_$v.log 2>&1
  echo "CARVEOUT=$v $c $(grep 'timeline\]' gpurun_out/ab2_${c}_$v.log | tail -1)" >> gpurun_out/ab2.txt
done; done
