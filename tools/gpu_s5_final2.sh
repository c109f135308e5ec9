# session-5 final evidence at HEAD: full GPU suite, smoke, default bench (both arms), launch list, ncu --set full of the c5 kernel
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s5_gpu_tests_final.txt 2>&1; echo rc=$?; tail -3 gpurun_out/s5_gpu_tests_final.txt
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/s5_bench_default.json 2> gpurun_out/s5_bench_default.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5_bench_reference.json 2> gpurun_out/s5_bench_reference.err; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/s5_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-heat-bath > gpurun_out/s5_ncu_l.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_c5_rounds -s 1 -c 1 -o gpurun_out/s5_c5_full2 -f python bench.py --rounds 100 --steps 1 --warmup 1 --no-cpu-baseline --no-heat-bath > gpurun_out/s5_ncu_c5b.log 2>&1; echo rc=$?
for n in 16384 65536 262144 524288; do timeout 300 python bench.py --n $n --steps 5 --rounds 400 --no-cpu-baseline --no-heat-bath 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': $n, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'kernel': d['roofline']['kernel'], 'frac': d['roofline']['frac']}))"; done > gpurun_out/s5_c5_sizes2.json 2>&1
tail -c 1500 gpurun_out/s5_bench_default.json
