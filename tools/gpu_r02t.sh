#!/bin/bash
# Checkpoint of the tree with RED rounds / dual prep streams / warp MT twist: GPU tests, smoke,
# every config at full size (parity_full_size + cpu_baseline), c2 reference arm, launch list, ncu of the chunk kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in c2 c1 c3 c4 c5; do
  timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c2_reference_arm.json 2> gpurun_out/bench_c2_ref.err
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_plain.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2400 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
CONFIGS="c2 c3" bash tools/gpu_ncu_chunk.sh
