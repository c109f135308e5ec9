# A/B of two engine builds on the same box: tools/ab.sh <bench args...>
# A = paper_2506_14781_b200/libtempergrid_b200.so, B = ..._ab.so (alternating runs)
for rep in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export TG_ENGINE_LIB=$PWD/paper_2506_14781_b200/libtempergrid_b200_ab.so; else unset TG_ENGINE_LIB; fi
    timeout 300 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4e' % d['value'], round(d['ms_per_step'], 3))"
  done
done
