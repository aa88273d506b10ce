#!/bin/bash
# wide-row pre-screen: parity tests, then c5 / c4 bench lines (no CPU leg)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big_means.py -x -q -k "wide_rows or configs_bitwise" > gpurun_out/wide_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/wide_pytest.log
for c in c5 c4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/wide_bench_$c.json 2> gpurun_out/wide_bench_$c.err
done
