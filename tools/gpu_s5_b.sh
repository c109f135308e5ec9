# session 5: cl chain deferral (A = new, B = before) and FLOAT dynamic item scheduling (TG_SF_DYN=0 = static)
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cl.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/s5_tests_clq.txt 2>&1; echo rc=$?; tail -3 gpurun_out/s5_tests_clq.txt
for n in 16384 65536 262144; do bash tools/ab.sh noclq --rounds 400 --n $n > gpurun_out/s5_ab_clq_$n.txt 2>&1; grep -E "^[AB] " gpurun_out/s5_ab_clq_$n.txt; done
bash tools/ab.sh noclq --rounds 400 --n 65536 --rule heat_bath > gpurun_out/s5_ab_clq_hb.txt 2>&1; grep -E "^[AB] " gpurun_out/s5_ab_clq_hb.txt
timeout 900 python -m pytest tests/test_gpu_float.py tests/test_gpu_stats.py tests/test_gpu_batch.py tests/test_gpu_configs.py tests/test_gpu_checkpoint.py -m gpu -x -q > gpurun_out/s5_tests_dyn.txt 2>&1; echo rc=$?; tail -3 gpurun_out/s5_tests_dyn.txt
for wl in c4 c3 c2; do for rep in 1 2; do for dynv in 1 0; do
  TG_SF_DYN=$dynv timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --rounds 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl dyn=$dynv', '%.4e' % d['value'], round(d['ms_per_step'], 3), d['roofline']['kernel'])"
done; done; done > gpurun_out/s5_ab_dyn.txt 2>&1; cat gpurun_out/s5_ab_dyn.txt
