#!/bin/bash
# usage: tools/gpu_profile.sh <config> <tag> [bench|nobench]   (on the GPU box, repo root)
CFG=${1:-C2}; TAG=${2:-r1}; MODE=${3:-bench}
mkdir -p gpurun_out
if [ "$MODE" = "bench" ]; then
  timeout 300 python bench.py --config $CFG --steps 1000 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_${CFG}_${TAG}.log 2>&1
fi
CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu"
KRE='regex:stream|compress_kernel|update_kernel|nccl'
timeout 300 $CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KRE" -s 9 -c 12 --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_${CFG}_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "$KRE" -s 9 -c 3 -o gpurun_out/prof_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo done
