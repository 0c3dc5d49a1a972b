#!/bin/bash
# Measured (not modeled) effect of the size threshold at N ranks over NVLink: 0 B vs 1 MiB.
# usage: gpu_threshold_multi.sh [N] [CONFIG]
N=${1:-4}
C=${2:-C2}
mkdir -p gpurun_out
for th in 0 1048576; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $N --steps 200 --warmup 5 --threshold-bytes $th --config $C --no-e2e > gpurun_out/thr_${C}_n${N}_$th.log 2>&1; echo th$th=$?
  grep '^{' gpurun_out/thr_${C}_n${N}_$th.log | tail -1
done
