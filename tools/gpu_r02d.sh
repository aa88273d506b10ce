#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3 c1; do
  BM_CHUNK_DBG=1 timeout 300 python tools/chunk_prof.py $c 20 > gpurun_out/dbg_$c.log 2>&1
done
