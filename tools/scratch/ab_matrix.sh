# A/B matrix on one box: LIBS="name=path ..." x ENVS (arguments; "" = defaults), two repetitions
for rep in 1 2; do
for l in ${LIBS:-main=paper_2410_22254_b200/_lib/libtlk.so}; do
for e in "$@"; do
  env TLK_LIB=$PWD/${l#*=} $e python bench.py --workload ${W:-cnn} --no-baselines --no-sweep --steps ${N:-200} --warmup 10 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${l%%=*} [$e]', round(d['value']), round(d['ms_per_step'],4), round((d.get('e2e') or {}).get('value') or 0))"
done; done; done
