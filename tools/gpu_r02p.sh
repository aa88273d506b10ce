#!/bin/bash
# RED rounds with the smaller shared-memory layout: timing, phases, source-level ncu of the chunk kernel.
mkdir -p gpurun_out
timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red.log 2>&1
BM_CHUNK_DBG=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_dbg.log 2>&1
BM_TIMELINE=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_tl.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "modes_agree" > gpurun_out/t_modes.log 2>&1; echo "rc=$?" >> gpurun_out/t_modes.log
timeout -s KILL 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c2_nocpu.json 2> gpurun_out/bench_c2.err
CONFIGS=c2 bash tools/gpu_ncu_chunk.sh
