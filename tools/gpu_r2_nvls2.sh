#!/bin/bash
# 2-GPU pass for the NVLS multicast pull: in-process group test, multi-process
# parity (p2p / nccl / nvls, eager and graph), N=2 bench lines p2p vs nvls.
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/nv2
timeout 600 python -m pytest tests/test_gpu_nvls.py -x -q -rs > ${O}_nvls_pytest.log 2>&1; echo nvls_pytest=$?; tail -5 ${O}_nvls_pytest.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -k "2-" > ${O}_multi_pytest.log 2>&1; echo multi_pytest=$?; tail -5 ${O}_multi_pytest.log
port=29670
for ex in nvls p2p; do
for c in C5 C2 C4; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --config $c --exchange $ex --steps 200 --warmup 10 --no-cpu --no-e2e > ${O}_bench_${c}_$ex.json 2> ${O}_bench_${c}_$ex.err
  echo "$c $ex rc=$?"
  tail -1 ${O}_bench_${c}_$ex.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['config']['exchange'], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})" 2>/dev/null
done
done
