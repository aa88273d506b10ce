#!/bin/bash
# cooperative vs plain launch of the chunk kernel (gap between chunk kernels)
mkdir -p gpurun_out
timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_coop.log 2>&1
BM_CHUNK_COOP=0 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_nocoop.log 2>&1
BM_CHUNK_COOP=0 timeout -s KILL 300 python tools/chunk_prof.py c3 > gpurun_out/prof_nocoop_c3.log 2>&1
timeout -s KILL 300 python tools/chunk_prof.py c3 > gpurun_out/prof_coop_c3.log 2>&1
BM_CHUNK_COOP=0 timeout -s KILL 300 python tools/chunk_prof.py c1 > gpurun_out/prof_nocoop_c1.log 2>&1
timeout -s KILL 300 python tools/chunk_prof.py c1 > gpurun_out/prof_coop_c1.log 2>&1
