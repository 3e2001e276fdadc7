python -m pytest tests/test_gpu_gpt.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in "TLK_GEMM_BN128=1" "TLK_GEMM_BN128=0"; do
for w in gpt xformer; do
env $v python bench.py --workload $w --no-baselines --no-sweep --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $v', round(d['value']), round(d['ms_per_step'],4))"
done; done; done
