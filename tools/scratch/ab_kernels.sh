# per-kernel warm times (bench.py's event-timed profile step) for several libtlk builds
for lib in ${LIBS:-paper_2410_22254_b200/_lib/libtlk.so}; do
  TLK_LIB=$lib python bench.py --workload ${W:-cnn} --no-baselines --no-sweep --steps 100 --warmup 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('== $lib', round(d['value']), round(d['ms_per_step'],4))
t=d.get('kernels') or {}
for n,v in sorted(t.items(), key=lambda x:-x[1]): print(f'  {n:24s} {v*1e3:9.2f} us')"
done
