# templated-kernel captures by launch index (ncu -k regex:<base name> -s <index>)
F="--set full --clock-control none --import-source on"
cap() {  # name regex skip command...
  local n=$1 r=$2 s=$3; shift 3
  ncu $F -k "regex:$r" -s $s -c 1 -o /tmp/$n -f "$@" > /dev/null 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/raw_$n.csv 2>/dev/null
}
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
cap c_conv2_fwd conv2_tc_kernel 10 $B
R="python tools/pack_step.py resnet18 8 128 1"
cap r_fwd_l1_halo tgemm 0 $R
cap r_dgrad_l1_halo tgemm 50 $R
cap r_wgrad_l1_tg tgemm 49 $R
cap r_dgrad_bn256 tgemm 20 $R
G="python tools/pack_step.py gpt 16 64 1"
cap g_scores tgemm 1 $G
cap g_fc tgemm 4 $G
