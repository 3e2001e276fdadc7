#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines of every workload
# (with CPU / K-process baselines) and ncu launch lists; outputs in gpurun_out/.
mkdir -p gpurun_out
T=${BENCH_TIMEOUT:-600}
for w in ${WORKLOADS:-cnn mlp resnet18 xformer gpt mix}; do
  timeout $T python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1
  echo "$w rc=$?" >> gpurun_out/bench_rc.txt
  tail -1 gpurun_out/bench_$w.log > gpurun_out/bench_$w.json
done
if [ -z "$NO_REF" ]; then
  timeout $T python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
  tail -1 gpurun_out/bench_reference.log > gpurun_out/bench_reference.json
fi
if [ -n "$LAUNCHES" ]; then
  M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
  timeout 300 ncu $M --log-file gpurun_out/launches_cnn.csv python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1 > /dev/null 2>&1
  for m in "mlp 4 64" "resnet18 8 128" "gpt 16 64" "xformer 32 32"; do
    set -- $m
    timeout 300 ncu $M --log-file gpurun_out/launches_$1.csv python tools/pack_step.py $1 $2 $3 1 > /dev/null 2>&1
  done
fi
ls gpurun_out
