# quick GPU check: parity tests of the touched packs, bench lines, ncu launch lists
T=${TESTS:-tests/test_gpu_pack.py tests/test_gpu_packed_backend.py tests/test_gpu_kernels.py tests/test_gpu_resnet.py}
python -m pytest $T -x -q 2>&1 | tail -3
for w in ${WORKLOADS:-cnn resnet18}; do
  n=200; [ $w = resnet18 -o $w = gpt ] && n=20
  python bench.py --workload $w --no-baselines --no-sweep --steps $n --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), round(d['ms_per_step'],4), (d.get('e2e') or {}).get('value'))"
done
if [ -n "$NCU" ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cnn.csv python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/launches_cnn.csv
fi
