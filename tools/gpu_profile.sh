# Round-end evidence capture (run on the GPU box from the repo root):
#   bash tools/gpu_profile.sh
# bench lines (default = the metric's config with the CPU baseline; c4 / c3 slot
# workloads), the launch list of the default bench, ncu --set full captures of
# the dominant kernels.  Each ncu run only after the same command exited 0.
set -x
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --rounds 20 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; echo rc=$?
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --rounds 50 > gpurun_out/bench_c3.json 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_tpw_rounds -s 1 -c 1 -o gpurun_out/plane_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_p.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slot2_sweep -s 3 -c 1 -o gpurun_out/slot2_c3 -f python bench.py --workload c3 --steps 1 --warmup 1 --rounds 5 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo rc=$?
ls -la gpurun_out
