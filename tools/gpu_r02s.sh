#!/bin/bash
# fused centroid pass in RED rounds, one event per chunk kernel, clock sampler before warm-up
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_core.py tests/test_gpu_big_means.py -x -q -m gpu > gpurun_out/t_quick.log 2>&1; echo "rc=$?" >> gpurun_out/t_quick.log
timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red.log 2>&1
BM_CHUNK_DBG=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_dbg.log 2>&1
timeout -s KILL 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2_nocpu.json 2> gpurun_out/bench_c2.err
