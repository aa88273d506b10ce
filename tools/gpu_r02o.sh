#!/bin/bash
# RED-delta exact-sum rounds (one grid barrier per round): quick parity, A/B timing, phases.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "modes_agree or tc_screen" > gpurun_out/t_modes.log 2>&1; echo "rc=$?" >> gpurun_out/t_modes.log
timeout -s KILL 900 python -m pytest tests/test_gpu_big_means.py -x -q -m gpu > gpurun_out/t_bm.log 2>&1; echo "rc=$?" >> gpurun_out/t_bm.log
timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red.log 2>&1
BM_CHUNK_RED=0 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_old.log 2>&1
BM_CHUNK_DBG=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_dbg.log 2>&1
timeout -s KILL 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
