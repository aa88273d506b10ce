# End-of-round artefacts: GPU tests, bench line (N=1, c2) + reference arm, the
# other configs' lines (parity cases, recorded for the notes), launch list of
# the host-driven loop and ncu --set full of the round assignment, update and
# streaming final pass.  Outputs in gpurun_out/.
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.err
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
export BM_GRAPHS=0
python tools/prof_assign.py c2 20 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_20chunks_hostloop.csv python tools/prof_assign.py c2 20 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_assign.py c2 3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assign_tma|k_final|k_update" -s 3 -c 8 -o gpurun_out/prof_round python tools/prof_assign.py c2 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
