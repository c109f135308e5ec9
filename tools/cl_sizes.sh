# Config-5 size sweep of the plane_cl kernel modes against plane_c5 (bench lines -> gpurun_out/cl_sizes.txt)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; : > gpurun_out/cl_sizes.txt
run() {  # label, env...
  label=$1; shift
  for n in ${SIZES:-16384 32768 65536 131072 262144 524288 1048576}; do
    env "$@" timeout 200 python bench.py --no-cpu-baseline --no-heat-bath --n $n --rounds $(( n >= 262144 ? 100 : 200 )) --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['config']['n_spins'], '%.3e'%d['value'], d['roofline']['kernel'], round(d['ms_per_step']*1000/d['config']['rounds_per_step'],2))" | tee -a gpurun_out/cl_sizes.txt
  done
}
for m in ${MODES:-cluster group1 group2 c5}; do
  case $m in
    cluster) run cluster TG_PLANE_CL=1 TG_PLANE_CL_MODE=cluster ;;
    group1) run group1 TG_PLANE_CL=1 TG_PLANE_CL_MODE=group TG_PLANE_CL_PAIR=0 ;;
    group2) run group2 TG_PLANE_CL=1 TG_PLANE_CL_MODE=group ;;
    c5) run c5 TG_PLANE_CL=0 ;;
    auto) run auto TG_NONE=1 ;;
  esac
done
