#!/bin/bash
# ncu --set full of one k_wide_screen and one k_wide_recheck launch (c5 chunk loop)
mkdir -p gpurun_out
BM_GRAPHS=0 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:'k_wide' -s 4 -c 2 -f -o gpurun_out/ncu_wide_c5 python tools/prof_assign.py c5 3 > gpurun_out/ncu_wide_c5.log 2>&1
