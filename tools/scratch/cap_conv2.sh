F="--set full --clock-control none --import-source on"
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
ncu $F -k "regex:conv2_tc_kernel" -s 10 -c 1 -o /tmp/c2f -f $B > /dev/null 2>&1
ncu -i /tmp/c2f.ncu-rep --page source --csv > gpurun_out/src_c2f.csv 2>/dev/null
ncu $F -k "regex:conv2_tc_kernel" -s 11 -c 1 -o /tmp/c2d -f $B > /dev/null 2>&1
ncu -i /tmp/c2d.ncu-rep --page source --csv > gpurun_out/src_c2d.csv 2>/dev/null
ncu -i /tmp/c2d.ncu-rep --page raw --csv > gpurun_out/raw_c2d.csv 2>/dev/null
