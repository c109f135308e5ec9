# A/B of two engine builds on the same box: tools/ab.sh NAME [bench args...]
# A = paper_2506_14781_b200/libtempergrid_b200.so, B = ..._NAME.so (alternating runs)
name=$1; shift
for rep in 1 2 3; do
  for v in A B; do
    if [ $v = B ]; then export TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_$name.so; else unset TG_ENGINE_LIB; fi
    timeout 300 python bench.py --no-cpu-baseline --no-heat-bath --steps 5 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $name', '%.4e' % d['value'], round(d['ms_per_step'], 3), d['roofline']['kernel'])"
  done
done
