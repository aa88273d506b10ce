#!/bin/bash
mkdir -p gpurun_out
for c in c1 c2; do BM_TIMELINE=2 timeout 300 python tools/chunk_prof.py $c 40 > gpurun_out/tl_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/chunk_prof.py c2 40 > gpurun_out/ncu_launch.log 2>&1
