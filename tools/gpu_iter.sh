#!/bin/bash
# One build -> measure iteration: GPU tests, chunk-kernel phase stamps and
# gaps for c1-c3, bench lines without the CPU leg.  Usage: bash tools/gpu_iter.sh [configs]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for c in ${PROF_CONFIGS:-c1 c2 c3}; do
  BM_CHUNK_DBG=1 timeout 300 python tools/chunk_prof.py $c 20 > gpurun_out/it_dbg_$c.log 2>&1
done
for c in ${BENCH_CONFIGS:-c2 c3}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/it_bench_$c.json 2> gpurun_out/it_bench_$c.err
done
