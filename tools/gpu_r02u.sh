#!/bin/bash
# RED as a template parameter (ordered instances without the red-mode code): c3/c1/c2 chunk kernel time, parity
mkdir -p gpurun_out
for c in c3 c1 c2; do timeout -s KILL 300 python tools/chunk_prof.py $c > gpurun_out/prof_$c.log 2>&1; done
BM_CHUNK_DBG=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_dbg.log 2>&1
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
