#!/bin/bash
# Measured (not modeled) effect of the size threshold at N ranks over NVLink: C2 at 0 B vs 1 MiB.
N=${1:-4}
mkdir -p gpurun_out
for th in 0 1048576; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $N --steps 200 --warmup 5 --threshold-bytes $th --no-e2e > gpurun_out/thr_n${N}_$th.log 2>&1; echo th$th=$?
  grep '^{' gpurun_out/thr_n${N}_$th.log | tail -1
done
