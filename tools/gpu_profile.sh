# Round profiling artefacts: GPU tests, bench line (N=1, c2), reference arm,
# launch list of a 20-chunk c2 run (graph mode), ncu --set full of the round
# assignment and the final pass.  Outputs in gpurun_out/.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.err
python tools/prof_assign.py c2 20 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_20chunks.csv python tools/prof_assign.py c2 20 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_assign.py c2 3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assign_tma|k_final" -s 6 -c 4 -o gpurun_out/prof_round python tools/prof_assign.py c2 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
