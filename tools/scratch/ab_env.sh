# A/B runtime switches on one box: each argument is an env assignment list ("" = defaults)
for rep in 1 2; do
for e in "$@"; do
  env $e python bench.py --workload ${W:-cnn} --no-baselines --no-sweep --steps ${N:-200} --warmup 10 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value']), round(d['ms_per_step'],4), (d.get('e2e') or {}).get('value'))"
done; done
