#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_big_means.py -x -q > gpurun_out/pt_multi.log 2>&1; echo "rc=$?" >> gpurun_out/pt_multi.log
for c in c2 c3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bf_$c.json 2> gpurun_out/bf_$c.err
done
