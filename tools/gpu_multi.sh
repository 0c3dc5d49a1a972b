#!/bin/bash
# multi-GPU checks on an N-GPU box: parity tests (NVLink peer-store and NCCL
# exchange), then the bench at N for each config with both transports
N=${1:-2}; TAG=${2:-r1}; CONFIGS=${3:-"C2 C5 C3 C4"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_pytest_${N}_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/multi_pytest_${N}_${TAG}.log
for c in $CONFIGS; do
  for x in p2p nccl; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 \
      bench.py --gpus $N --config $c --steps 200 --warmup 5 --no-cpu --exchange $x > gpurun_out/bench_${c}_n${N}_${x}_${TAG}.log 2>&1
  done
done
echo done
