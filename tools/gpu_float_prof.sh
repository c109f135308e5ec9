# FLOAT engine evidence: bench lines of configs 4 and 3, ncu --set full of slotf_sweep_kernel on each.
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --rounds 20 --no-cpu-baseline > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo rc=$?
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --rounds 20 --no-cpu-baseline > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slotf_sweep -s 3 -c 1 -o gpurun_out/slotf_c4 -f python bench.py --workload c4 --steps 1 --warmup 1 --rounds 5 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slotf_sweep -s 3 -c 1 -o gpurun_out/slotf_c3 -f python bench.py --workload c3 --steps 1 --warmup 1 --rounds 5 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/bench_c4.json; tail -c 600 gpurun_out/bench_c3.json
