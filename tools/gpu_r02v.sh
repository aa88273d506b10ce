#!/bin/bash
# Final tree of the round: GPU tests, smoke, c2 bench (parity + cpu baseline), reference arm, the other configs.
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c2_reference_arm.json 2> gpurun_out/bench_c2_ref.err
for c in c1 c3 c4 c5; do
  timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
BM_CHUNK_PDL=1 timeout -s KILL 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c2_pdl.json 2>&1
