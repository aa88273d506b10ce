#!/bin/bash
# persistent chunk kernel: parity first, then quick benches
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_big_means.py -x -q > gpurun_out/pt_bm.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bm.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for c in c2 c3 c1; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-e2e > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err
done
