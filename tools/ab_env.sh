# A/B of one engine build under two environments on the same box: tools/ab_env.sh VAR=VALUE [bench args...]
# A = default environment, B = with VAR=VALUE exported (alternating runs)
kv=$1; shift
for rep in 1 2 3; do
  for v in A B; do
    if [ $v = B ]; then export "$kv"; else unset "${kv%%=*}"; fi
    timeout 300 python bench.py --no-cpu-baseline --no-heat-bath --steps 5 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $kv', '%.4e' % d['value'], round(d['ms_per_step'], 3), d['roofline']['kernel'])"
  done
done
