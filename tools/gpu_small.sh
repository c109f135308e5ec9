# Small-N config-5 data: size sweep on the default kernel, stage timeline of the tpw profiling variant.
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/c5_sizes.sh
cat gpurun_out/c5_sizes.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['n_spins'], '%.3e'%d['value'], d['roofline']['kernel'], d['ms_per_step']*1000/d['config']['rounds_per_step'])"
for n in 16384 65536; do
TG_PLANE_C5=0 TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_P.so timeout 300 python tools/round_stages.py $n
done > gpurun_out/stages_small.txt 2>&1
cat gpurun_out/stages_small.txt
