#!/bin/bash
# ncu --set full captures of the round's top kernels (one GPU, serialised);
# raw CSV exported on the box for tools/ncu_summary.py / ncu_hot.py.
mkdir -p gpurun_out
F="--set full --clock-control none --import-source on"
cap() {  # name regex skip command...
  local n=$1 r=$2 s=$3; shift 3
  timeout 300 ncu $F -k "regex:$r" -s $s -c 1 -o gpurun_out/cap_$n -f "$@" > /dev/null 2>&1
}
B="python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1"
cap cnn_fc1_wgrad_adam fc1_wgrad_adam 5 $B
cap cnn_conv2_fwd conv2_tc_kernel 10 $B
cap cnn_conv1_fwd conv1_fwd 5 $B
cap cnn_conv1_wgrad conv1_wgrad 5 $B
cap cnn_head cnn_head 5 $B
cap mlp_step mlp_step 2 python tools/pack_step.py mlp 4 64 3
cap mlp_wgrad_adam mlp_wgrad 2 python tools/pack_step.py mlp 4 64 3
cap gpt_attn_fwd attn_fwd 1 python tools/pack_step.py gpt 16 64 1
cap gpt_attn_bwd attn_bwd 1 python tools/pack_step.py gpt 16 64 1
cap xf_attn_fwd attn_fwd 1 python tools/pack_step.py xformer 32 32 1
cap xf_attn_bwd attn_bwd 1 python tools/pack_step.py xformer 32 32 1
# tiny-GPT dense GEMMs (launch order of one step: qkv, proj, fc, fc2 per layer;
# backward of the last layer after the 24 forward + 3 head GEMMs)
cap gpt_gemm_qkv tgemm 0 python tools/pack_step.py gpt 16 64 1
cap gpt_gemm_fc tgemm 2 python tools/pack_step.py gpt 16 64 1
cap gpt_gemm_fc2 tgemm 3 python tools/pack_step.py gpt 16 64 1
cap gpt_gemm_fc2_wgrad tgemm 27 python tools/pack_step.py gpt 16 64 1
cap gpt_gemm_fc2_dgrad tgemm 28 python tools/pack_step.py gpt 16 64 1
cap gpt_gemm_fc_dgrad tgemm 30 python tools/pack_step.py gpt 16 64 1
ls gpurun_out/cap_*
