#!/bin/bash
# phase stamps of the persistent chunk kernel (CTA 0, globaltimer) for c1-c3
mkdir -p gpurun_out
for c in c1 c2 c3; do
  BM_CHUNK_DBG=1 timeout 300 python tools/chunk_prof.py $c 20 > gpurun_out/dbg_$c.log 2>&1
done
