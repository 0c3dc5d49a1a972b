#!/bin/bash
# experiment: fused pull variants (BPC_PULL_MODE 0/1/2) at N=2, plus the 1-GPU A/B
mkdir -p gpurun_out
CONFIGS="C2 C5" bash tools/ab_bench.sh
for m in 2 1 0; do
  BPC_PULL_MODE=$m timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "p2p and 2" > gpurun_out/pm_pytest_$m.log 2>&1; echo rc=$? >> gpurun_out/pm_pytest_$m.log
  for c in C2 C5 C4; do
    BPC_PULL_MODE=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
      bench.py --gpus 2 --config $c --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/pm_${c}_$m.log 2>&1
  done
done
