#!/bin/bash
# Final weak-scaling pass on N GPUs: multi-GPU parity (p2p / nccl / nvls, eager / graph)
# and bench lines with the default exchange (auto) for C2-C5, plus the explicit
# p2p / nvls variants of C5.
N=${1:-4}
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out/scale
O=gpurun_out/scale/n$N
nvidia-smi -L > ${O}_gpus.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_nvls.py -x -q -rs -k "$N- or nvls_local" > ${O}_pytest.log 2>&1; echo pytest=$?; tail -3 ${O}_pytest.log
port=29800
for spec in C5:auto C2:auto C3:auto C4:auto C5:p2p C5:nvls; do
  IFS=: read c ex <<< "$spec"
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --exchange $ex --no-cpu --no-e2e > ${O}_bench_${c}_$ex.json 2> ${O}_bench_${c}_$ex.err
  echo "$c $ex rc=$?"
  tail -1 ${O}_bench_${c}_$ex.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['config']['exchange'], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})" 2>/dev/null
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((port+1)) bench.py --gpus $N > ${O}_bench_default.json 2> ${O}_bench_default.err; echo "default rc=$?"
tail -1 ${O}_bench_default.json | head -c 400
