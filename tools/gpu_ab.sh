#!/bin/bash
mkdir -p gpurun_out
for v in A B A B; do for c in c2 c3; do
  if [ $v = A ]; then L=$PWD/_ab/paper_2204_07485_b200/_lib/libbigmeans_b200.so; else L=""; fi
  BM_LIB_PATH=$L BM_CHUNK_FIX=0 timeout 300 python tools/chunk_prof.py $c 40 > gpurun_out/ab_${c}_$v.log 2>&1
  echo "$v $c $(tail -1 gpurun_out/ab_${c}_$v.log)" >> gpurun_out/ab.txt
done; done
