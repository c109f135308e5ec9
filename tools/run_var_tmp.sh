mkdir -p gpurun_out; rm -f gpurun_out/var.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_paths.py -x -q > gpurun_out/par.log 2>&1; echo par_rc=$? >> gpurun_out/par.log
for v in A D E O; do
  case $v in A) unset TG_ENGINE_LIB; unset TG_PLANE_TPW;; B|C|D|E) export TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_$v.so;; O) unset TG_ENGINE_LIB; export TG_PLANE_TPW=0;; esac
  timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4e' % d['value'], round(d['ms_per_step'], 3), '%.3e'%d['e2e']['value'])" >> gpurun_out/var.log 2>&1
done
unset TG_ENGINE_LIB; unset TG_PLANE_TPW
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_tpw -s 1 -c 1 -o gpurun_out/tpw12 -f python bench.py --steps 1 --warmup 1 --rounds 20 --no-cpu-baseline > gpurun_out/ncu_t.log 2>&1
