#!/bin/bash
# usage: tools/gpu_profile.sh <config> <tag> <launches|full> [kernel-regex] [count]
# (on the GPU box, repo root).  One ncu tool per call: the plain command runs
# first and must exit 0.
CFG=${1:-C2}; TAG=${2:-r1}; MODE=${3:-full}; KRE=${4:-'regex:stream|compress_kernel|update_kernel|p2p|nccl'}; CNT=${5:-3}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
if [ "$MODE" = "launches" ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KRE" -s 9 -c 12 --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_${CFG}_${TAG}.log 2>&1
else
  ncu --set full --clock-control none --import-source on -k "$KRE" -s 9 -c $CNT -o gpurun_out/prof_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
fi
echo done
