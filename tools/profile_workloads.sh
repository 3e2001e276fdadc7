#!/bin/bash
# ncu evidence for the transformer and ResNet packs (run under gpurun, 1 GPU).
# Launch lists (every kernel of one step) + full-set captures of the top
# kernels, exported to CSV on the box (the .ncu-rep files stay in /tmp).
set -x
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum --clock-control none --csv"
[ -n "$NOLAUNCH" ] || ncu $M --log-file gpurun_out/launches_gpt.csv python tools/pack_step.py gpt 16 64 1 > /dev/null 2>&1
[ -n "$NOLAUNCH" ] || ncu $M --log-file gpurun_out/launches_resnet18.csv python tools/pack_step.py resnet18 8 128 1 > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
# tgemm launch order in one step (see csrc/gpt.cu, csrc/resnet.cu):
#   GPT: per layer qkv, scores, pv, proj, fc, fc2 (x6), head_ce, head_dgrad,
#        head_wgrad, then per layer fc2_wgrad, fc2_dgrad, ..., attn_dp (+6) ...
#   ResNet: 19 forward convs (l1.0 c1 = 0, l2.0 c2 = 5), then per block in
#        reverse wgrad c2, dgrad c2, wgrad c1, dgrad c1 [, wgrad ds, dgrad ds]
cap() {  # name model lanes batch skip
  ncu $F -k regex:tgemm -s $5 -c 1 -o /tmp/$1 -f python tools/pack_step.py $2 $3 $4 1 > /dev/null 2>&1
}
cap g_qkv gpt 16 64 0
cap g_scores gpt 16 64 1
cap g_fc gpt 16 64 4
cap g_fc2dgrad gpt 16 64 40
cap g_attndp gpt 16 64 45
cap r_fwd_l1 resnet18 8 128 0
cap r_fwd_l2 resnet18 8 128 5
cap r_wgrad_l3 resnet18 8 128 29
cap r_wgrad_l1 resnet18 8 128 49
cap r_dgrad_l1 resnet18 8 128 50
cap r_dgrad_l2 resnet18 8 128 40
ncu $F -k regex:rn_bn_bwd_apply -s 0 -c 1 -o /tmp/r_bnapply -f python tools/pack_step.py resnet18 8 128 1 > /dev/null 2>&1
for f in /tmp/g_*.ncu-rep /tmp/r_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv > gpurun_out/raw_$b.csv
  ncu -i $f --page source --csv > gpurun_out/src_$b.csv 2>/dev/null
done
ls -la gpurun_out
