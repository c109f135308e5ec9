mkdir -p gpurun_out; rm -f gpurun_out/var.log
for n in 4096 16384 65536 262144 1048576; do
  r=$(( n >= 262144 ? 100 : 1000 ))
  timeout 300 python bench.py --no-cpu-baseline --n $n --rounds $r --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, '%.4e' % d['value'], 'us/round %.2f' % (1000*d['ms_per_step']/$r))" >> gpurun_out/var.log 2>&1
done
