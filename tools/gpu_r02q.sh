#!/bin/bash
# Dual prep streams + single-warp MT twist + MMA issue beside the norms: parity, timing.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_search.py tests/test_gpu_core.py -x -q -m gpu > gpurun_out/t_quick.log 2>&1; echo "rc=$?" >> gpurun_out/t_quick.log
timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red.log 2>&1
BM_TIMELINE=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_tl.log 2>&1
BM_CHUNK_DBG=1 timeout -s KILL 300 python tools/chunk_prof.py c2 > gpurun_out/prof_red_dbg.log 2>&1
timeout -s KILL 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in c1 c3; do timeout -s KILL 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${c}_nocpu.json 2> gpurun_out/bench_$c.err; done
