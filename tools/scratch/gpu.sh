#!/bin/bash
# build libtlk here (fail fast), then run the given command on the B200 box
set -e
cd /root/repo
python -m paper_2410_22254_b200.build > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; exit 1; }
T=${GPU_TIMEOUT:-900}
/usr/local/graft/bin/gpurun --timeout $T -- "$@"
