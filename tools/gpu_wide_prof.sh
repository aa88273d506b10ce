#!/bin/bash
# Launch lists (per-kernel durations) of a few c4 / c5 chunks on the multi-launch (wide-row) path
mkdir -p gpurun_out
for c in ${WCONFIGS:-c4 c5}; do
  BM_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
    --log-file gpurun_out/wide_launch_$c.csv python tools/prof_assign.py $c 6 > gpurun_out/wide_launch_$c.log 2>&1
done
