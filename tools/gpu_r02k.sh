#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bk_$c.json 2> gpurun_out/bk_$c.err
done
BM_TIMELINE=1 timeout 300 python tools/chunk_prof.py c2 > gpurun_out/tl_c2.log 2>&1
