# one GPU round trip: GPU tests, then the c2 / c5 bench lines (no e2e / CPU arm)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for c in ${BENCH_CONFIGS:-c2}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -3 gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['step_breakdown_ms'])"
done
