#!/bin/bash
# Run tools/round_captures.sh, then summarise every capture ON THE BOX (the
# .ncu-rep files are too large to bring back as a set): gpurun_out/ncu_full.txt
# (tools/ncu_summary.py) and gpurun_out/ncu_hot_<name>.txt (top stall sites).
bash tools/round_captures.sh > gpurun_out/rc.log 2>&1
python tools/ncu_summary.py gpurun_out/cap_*.ncu-rep > gpurun_out/ncu_full.txt 2>&1
for f in gpurun_out/cap_*.ncu-rep; do
  n=$(basename $f .ncu-rep)
  python tools/ncu_hot.py $f 20 > gpurun_out/ncu_hot_${n#cap_}.txt 2>&1
done
mkdir -p gpurun_out/keep
for n in gpt_gemm_fc2_dgrad gpt_attn_fwd; do mv gpurun_out/cap_$n.ncu-rep gpurun_out/keep/ 2>/dev/null; done
rm -f gpurun_out/cap_*.ncu-rep
du -sh gpurun_out
