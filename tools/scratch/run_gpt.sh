python -m pytest tests/test_gpu_gpt.py -q -x 2>&1 | tail -2
for w in gpt xformer; do
python bench.py --workload $w --no-baselines --no-sweep --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), round(d['ms_per_step'],4))
t=d.get('kernels') or {}
tot=sum(t.values())
for n,v in sorted(t.items(), key=lambda x:-x[1])[:12]: print(f'  {n:24s} {v*1e3:9.1f} us {100*v/tot:5.1f}%')"
done
