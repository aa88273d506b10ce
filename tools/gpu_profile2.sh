# ncu artefacts on the host-driven chunk loop (BM_GRAPHS=0: ncu does not profile
# kernel nodes of graphs that may set conditional handles)
set -x
export BM_GRAPHS=0
true && \
python tools/prof_assign.py c2 3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assign_tma|k_final|k_update" -s 3 -c 8 -o gpurun_out/prof_round python tools/prof_assign.py c2 3 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
