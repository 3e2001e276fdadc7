#!/bin/bash
# Bench lines of every workload on one B200 (run under gpurun); outputs in gpurun_out/.
mkdir -p gpurun_out
T=${BENCH_TIMEOUT:-600}
for w in ${WORKLOADS:-mlp resnet18 xformer gpt mix paper24}; do
  timeout $T python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1
  echo "$w rc=$?" >> gpurun_out/bench_rc.txt
  tail -1 gpurun_out/bench_$w.log > gpurun_out/bench_$w.json
done
timeout $T python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
tail -1 gpurun_out/bench_reference.log > gpurun_out/bench_reference.json
