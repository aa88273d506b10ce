#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big_means.py -x -q > gpurun_out/pt_bm.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bm.log
for c in c2 c3 c1; do
  timeout 300 python tools/chunk_prof.py $c 40 > gpurun_out/cp_$c.log 2>&1
  BM_CHUNK_DBG=1 timeout 300 python tools/chunk_prof.py $c 20 > gpurun_out/dbg_$c.log 2>&1
done
