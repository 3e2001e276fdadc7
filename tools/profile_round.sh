#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines of every
# workload (with CPU / K-process baselines), ncu launch lists (device time +
# DRAM bytes per kernel) and --set full captures of the top kernels, exported
# to CSV on the box.  Summarised into profiles/ by tools/make_round_profiles.py.
mkdir -p gpurun_out
for w in cnn mlp resnet18 xformer gpt; do
  python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1
  tail -1 gpurun_out/bench_$w.log > gpurun_out/bench_$w.json
done
python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
tail -1 gpurun_out/bench_reference.log > gpurun_out/bench_reference.json
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M --log-file gpurun_out/launches_cnn.csv python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1 > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_resnet18.csv python tools/pack_step.py resnet18 8 128 1 > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_gpt.csv python tools/pack_step.py gpt 16 64 1 > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
cap() {  # name regex skip command...
  local n=$1 r=$2 s=$3; shift 3
  ncu $F -k "regex:$r" -s $s -c 1 -o /tmp/$n -f "$@" > /dev/null 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/raw_$n.csv 2>/dev/null
}
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
cap c_fc1_wgrad_adam fc1_wgrad_adam 5 $B
cap c_conv2_fwd conv2_tc_kernel 10 $B
cap c_conv2_dgrad conv2_tc_kernel 11 $B
cap c_conv2_wgrad conv2_wgrad_tc 5 $B
cap c_fc1_dgrad tc_gemm_tma_kernel 5 $B
cap c_cnn_opt cnn_opt 5 $B
cap c_cnn_head cnn_head 5 $B
R="python tools/pack_step.py resnet18 8 128 1"
cap r_fwd_l1_halo tgemm 0 $R
cap r_dgrad_l1_halo tgemm 50 $R
cap r_wgrad_l1_tg tgemm 49 $R
cap r_dgrad_bn256 tgemm 20 $R
cap r_bn_bwd_apply rn_bn_bwd_apply 0 $R
G="python tools/pack_step.py gpt 16 64 1"
cap g_scores tgemm 1 $G
cap g_fc tgemm 4 $G
ls -la gpurun_out
