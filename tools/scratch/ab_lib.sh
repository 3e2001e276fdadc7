# A/B two libtlk builds on the same box: TLK_LIB=$A vs the in-tree build
A=${A:-_ab/base/libtlk.so}
for rep in 1 2 3; do
for lib in $A paper_2410_22254_b200/_lib/libtlk.so; do
  for w in ${WORKLOADS:-cnn}; do
    n=200; [ $w = resnet18 -o $w = gpt ] && n=20
    TLK_LIB=$lib python bench.py --workload $w --no-baselines --no-sweep --steps $n --warmup 10 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '$lib'[:20], round(d['value']), round(d['ms_per_step'],4), (d.get('e2e') or {}).get('value'))"
  done
done; done
