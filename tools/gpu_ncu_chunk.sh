#!/bin/bash
# ncu --set full of one persistent chunk kernel launch (not k_chunk_fix) per config
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3}; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:'k_chunk<' -s 3 -c 1 -f -o gpurun_out/ncu_chunk_$c python tools/chunk_prof.py $c 6 > gpurun_out/ncu_chunk_$c.log 2>&1
done
