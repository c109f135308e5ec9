# A/B of FLOAT-engine library variants on configs 4 and 3: tools/abfloat.sh NAME...
for wl in c4 c3; do
for rep in 1 2; do
  for v in A "$@"; do
    if [ $v = A ]; then unset TG_ENGINE_LIB; else export TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_$v.so; fi
    timeout 300 python bench.py --workload $wl --steps 3 --warmup 2 --rounds 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $v', '%.4e' % d['value'], round(d['ms_per_step'], 3), d['roofline']['kernel'])"
  done
done
done
