F="--set full --clock-control none --import-source on"
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
for k in conv1_wgrad conv1_fwd head_kernel cnn_opt; do
  ncu $F -k "regex:$k" -s 5 -c 1 -o /tmp/c_$k -f $B > /dev/null 2>&1
  ncu -i /tmp/c_$k.ncu-rep --page raw --csv > gpurun_out/raw_c_$k.csv 2>/dev/null
  ncu -i /tmp/c_$k.ncu-rep --page source --csv > gpurun_out/src_c_$k.csv 2>/dev/null
done
ls -la gpurun_out | tail -8
