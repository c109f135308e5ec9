# session-5 A/B: compare8 (LSB-first 8-plane prefix, one-instruction selects) + 32-bit row offsets vs the old build
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_c5.py tests/test_gpu_cl.py tests/test_gpu_tpw.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s5_tests_cmp8.txt 2>&1; echo rc=$?; tail -3 gpurun_out/s5_tests_cmp8.txt
bash tools/ab.sh old --rounds 400 > gpurun_out/s5_ab_n20.txt 2>&1; cat gpurun_out/s5_ab_n20.txt
bash tools/ab.sh old --rounds 400 --rule heat_bath > gpurun_out/s5_ab_n20_hb.txt 2>&1; cat gpurun_out/s5_ab_n20_hb.txt
bash tools/ab.sh old --rounds 400 --n 65536 > gpurun_out/s5_ab_n16.txt 2>&1; cat gpurun_out/s5_ab_n16.txt
bash tools/ab.sh old --rounds 400 --n 16384 > gpurun_out/s5_ab_n14.txt 2>&1; cat gpurun_out/s5_ab_n14.txt
bash tools/ab.sh old --rounds 400 --n 262144 > gpurun_out/s5_ab_n18.txt 2>&1; cat gpurun_out/s5_ab_n18.txt
