#!/bin/bash
# ncu --set full of the multi-launch assignment kernel on the wide-row configs (c4: k_assign_tma;
# c5: k_assign_tma in pre-screened mode + the k_wide_* kernels), host-driven loop so that ncu sees every kernel
mkdir -p gpurun_out
for c in c4 c5; do
  BM_GRAPHS=0 timeout 600 python tools/prof_assign.py $c 3 > gpurun_out/plain_$c.log 2>&1 && \
  BM_GRAPHS=0 timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:'k_assign_tma|k_wide' -s 8 -c 6 -f -o gpurun_out/ncu_assign_$c python tools/prof_assign.py $c 3 > gpurun_out/ncu_assign_$c.log 2>&1
  ncu -i gpurun_out/ncu_assign_$c.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/ncu_assign_$c.csv 2>&1
  rm -f gpurun_out/ncu_assign_$c.ncu-rep
done
