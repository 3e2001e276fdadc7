# round-2 closing evidence (after the conv1 fwd change): GPU tests, CNN bench line + reference arm, CNN launch list, timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
WORKLOADS="cnn" LAUNCHES= bash tools/round_benches.sh
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 300 ncu $M --log-file gpurun_out/launches_cnn.csv python bench.py --steps 3 --warmup 3 --no-baselines --no-sweep --profile-iters 1 > /dev/null 2>&1
TLK_LIB=$PWD/_ab/kt/libtlk.so python tools/cnn_timeline.py 8 6 > gpurun_out/timeline_defer.txt 2>&1
ls gpurun_out
