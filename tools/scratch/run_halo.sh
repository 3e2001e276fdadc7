python -m pytest tests/test_gpu_resnet.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for v in "TLK_CONV_BN256=0" "TLK_CONV_BN256=1"; do
env $v python bench.py --workload resnet18 --no-baselines --no-sweep --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('resnet $v', round(d['value']), round(d['ms_per_step'],4))"
done; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_resnet18.csv python tools/pack_step.py resnet18 8 128 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_resnet18.csv
