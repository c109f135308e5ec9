# Round-2 final evidence: default bench (both arms), launch list, ncu --set full of plane_cl at 2^16 and 2^14.
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-heat-bath > gpurun_out/ncu_l.log 2>&1; echo rc=$?
timeout 600 python bench.py --n 65536 --steps 5 --no-cpu-baseline > gpurun_out/bench_n16.json 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_cl_rounds -s 1 -c 1 -o gpurun_out/cl_n16 -f python bench.py --n 65536 --rounds 400 --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/ncu_cl16.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_cl_rounds -s 1 -c 1 -o gpurun_out/cl_n14 -f python bench.py --n 16384 --rounds 400 --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/ncu_cl14.log 2>&1; echo rc=$?
tail -c 400 gpurun_out/bench_default.json
