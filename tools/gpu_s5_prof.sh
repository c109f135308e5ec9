# session-5 profiles: ncu --set full of plane_c5_rounds_kernel (100 rounds per launch) and of slotf_sweep_kernel (config 4)
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --rounds 100 --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/s5_prof_pre.json 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_c5_rounds -s 1 -c 1 -o gpurun_out/s5_c5_full -f python bench.py --rounds 100 --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/s5_ncu_c5.log 2>&1; echo rc=$?
timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --rounds 5 --no-cpu-baseline > gpurun_out/s5_prof_c4_pre.json 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slotf_sweep -s 3 -c 1 -o gpurun_out/s5_slotf_c4 -f python bench.py --workload c4 --steps 1 --warmup 1 --rounds 5 --no-cpu-baseline > gpurun_out/s5_ncu_c4.log 2>&1; echo rc=$?
