#!/bin/bash
# 4-GPU pass: parity (p2p / nccl / nvls x eager / graph) and weak-scaling bench lines.
N=${1:-4}
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/m$N
nvidia-smi -L > ${O}_gpus.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -k "$N-" > ${O}_pytest.log 2>&1; echo pytest=$?; tail -3 ${O}_pytest.log
timeout 300 python -m pytest tests/test_gpu_nvls.py -x -q -rs > ${O}_nvls_pytest.log 2>&1; echo nvls_pytest=$?; tail -2 ${O}_nvls_pytest.log
port=29710
for spec in C5:nvls C5:p2p C2:nvls C2:p2p C4:nvls C4:p2p C3:p2p C5:nccl; do
  IFS=: read c ex <<< "$spec"
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --exchange $ex --steps 200 --warmup 10 --no-cpu --no-e2e > ${O}_bench_${c}_$ex.json 2> ${O}_bench_${c}_$ex.err
  echo "$c $ex rc=$?"
  tail -1 ${O}_bench_${c}_$ex.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['config']['exchange'], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d.get('bus'))" 2>/dev/null
done
