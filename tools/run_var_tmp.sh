mkdir -p gpurun_out; rm -f gpurun_out/var.log
run() { timeout 300 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', '%.4e' % d['value'], d['roofline']['kernel'])" >> gpurun_out/var.log 2>&1; }
export V="metro tpw-generic"; TG_PLANE_FAST=0 run
export V="metro old-generic"; TG_PLANE_FAST=0 TG_PLANE_TPW=0 run
export V="metro old-fast"; TG_PLANE_TPW=0 run
export V="hb tpw-generic"; run --rule heat_bath
export V="hb old-fast"; TG_PLANE_TPW=0 run --rule heat_bath
export V="hb old-generic"; TG_PLANE_FAST=0 TG_PLANE_TPW=0 run --rule heat_bath
export V="metro n2^16 tpw"; run --n 65536 --rounds 500
export V="metro n2^16 old"; TG_PLANE_TPW=0 run --n 65536 --rounds 500
