#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_chunk -s 3 -c 1 -f -o gpurun_out/ncu_chunk_$c python tools/chunk_prof.py $c 6 > gpurun_out/ncu_chunk_$c.log 2>&1
done
