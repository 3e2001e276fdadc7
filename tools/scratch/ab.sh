#!/bin/bash
# A/B of libtlk builds: VARIANTS="name=path ..." WORKLOADS="gpt ..." bash tools/scratch/ab.sh
mkdir -p gpurun_out
for w in ${WORKLOADS:-gpt}; do
  for v in ${VARIANTS:-main=paper_2410_22254_b200/_lib/libtlk.so}; do
    n=${v%%=*}; l=${v#*=}
    TLK_LIB=$PWD/$l timeout 400 python bench.py --workload $w --no-baselines --no-sweep > gpurun_out/ab_${w}_$n.log 2>&1
    tail -1 gpurun_out/ab_${w}_$n.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d.get('kernels',{})
  top=sorted(k.items(),key=lambda x:-x[1])[:6]
  print('$w $n', round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], ' '.join(f'{a}={b:.3f}' for a,b in top))
except Exception as e: print('$w $n FAIL', e)"
  done
done
