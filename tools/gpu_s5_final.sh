# session-5 final evidence: full GPU suite, default bench (both arms), launch list, size sweep, float configs
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s5_gpu_tests_final.txt 2>&1; echo rc=$?; tail -3 gpurun_out/s5_gpu_tests_final.txt
timeout 900 python bench.py > gpurun_out/s5_bench_default.json 2> gpurun_out/s5_bench_default.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5_bench_reference.json 2> gpurun_out/s5_bench_reference.err; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/s5_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-heat-bath > gpurun_out/s5_ncu_l.log 2>&1; echo rc=$?
for n in 16384 32768 65536 131072 262144 524288 1048576; do timeout 300 python bench.py --n $n --steps 5 --rounds 400 --no-cpu-baseline --no-heat-bath 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': $n, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'kernel': d['roofline']['kernel'], 'frac': d['roofline']['frac']}))"; done > gpurun_out/s5_c5_sizes.json 2>&1; cat gpurun_out/s5_c5_sizes.json
for wl in c4 c3; do for rule in metropolis heat_bath; do timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --rounds 20 --rule $rule --no-cpu-baseline > gpurun_out/s5_bench_${wl}_${rule}.json 2>/dev/null; tail -c 300 gpurun_out/s5_bench_${wl}_${rule}.json; done; done
tail -c 1200 gpurun_out/s5_bench_default.json
