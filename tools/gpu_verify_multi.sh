#!/bin/bash
# Multi-GPU pass over HEAD on one box: the n-rank parity tests and an N-GPU bench line.
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_n$N.log 2>&1; echo pytest_multi=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 200 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_multi_n$N.log; grep '^{' gpurun_out/bench_n$N.log | tail -1
