#!/bin/bash
# ncu evidence for the CNN pack (run under gpurun, 1 GPU).  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
NCU=${NCU:-ncu}
# 1) launch list: every kernel of a short bench run with its device time
$NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-baselines --profile-iters 1 > gpurun_out/launches_bench.log 2>&1
# 2) full sets of the top kernels
for K in ${KERNELS:-conv2_tc_kernel conv2_wgrad_tc Fc1Dgrad optimizer_kernel}; do
  $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$K -s 3 -c ${NCU_COUNT:-1} \
       -o gpurun_out/prof_$K -f python bench.py --steps 3 --warmup 3 --no-baselines --profile-iters 1 > gpurun_out/prof_$K.log 2>&1
done
ls -la gpurun_out
