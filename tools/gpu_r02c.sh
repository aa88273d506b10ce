#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3 c1; do
  BM_TIMELINE=1 timeout 300 python tools/chunk_prof.py $c > gpurun_out/cp_$c.log 2>&1
  BM_PERSIST=0 BM_TIMELINE=1 timeout 300 python tools/chunk_prof.py $c > gpurun_out/cp0_$c.log 2>&1
done
