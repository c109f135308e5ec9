# Round-2 evidence capture: GPU tests, bench, launch list, ncu --set full of the c5 kernel.
set -x
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1; echo rc=$?; tail -3 gpurun_out/gputests.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-heat-bath > gpurun_out/ncu_l.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_c5_rounds -s 1 -c 1 -o gpurun_out/c5_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/ncu_p.log 2>&1; echo rc=$?
ls -la gpurun_out
