#!/bin/bash
# ncu --set full captures (kept under 64 MiB of gpurun_out): chunk kernel c2 / c3, wide kernels c5
mkdir -p gpurun_out
CONFIGS="${CONFIGS:-c2 c3}" bash tools/gpu_ncu_chunk.sh
bash tools/gpu_ncu_wide.sh
for f in gpurun_out/*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.csv 2>/dev/null; done
ls -la gpurun_out
