#!/bin/bash
# compute-sanitizer over the small engine cases (one tool per pass); logs -> gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in c2_small_tc c3_small_ffma c1_small_f64 wide_rows repairs; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py $c \
      > gpurun_out/san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" >> gpurun_out/san_summary.txt
  done
done
