# round-2 final evidence on one box: GPU tests, every workload's bench line, launch lists, CNN captures
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
LAUNCHES=1 bash tools/round_benches.sh
F="--set full --clock-control none --import-source on"
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
for k in "fc1_wgrad_adam fc1_wgrad_adam 5" "conv1_wgrad conv1_wgrad 5" "conv1_fwd conv1_fwd 5"; do
  set -- $k
  timeout 300 ncu $F -k "regex:$2" -s $3 -c 1 -o gpurun_out/cap_cnn_$1 -f $B > /dev/null 2>&1
done
ls gpurun_out
