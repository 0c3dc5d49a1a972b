#!/bin/bash
# NVLS pull variants at N=2: copy kernel (default) vs in-server multicast stores.
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/nv4
N=${1:-2}
timeout 600 python -m pytest tests/test_gpu_nvls.py -x -q -rs > ${O}_nvls_pytest.log 2>&1; echo nvls_pytest=$?; tail -2 ${O}_nvls_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "$N-nvls" > ${O}_multi_pytest.log 2>&1; echo multi_pytest=$?; tail -2 ${O}_multi_pytest.log
port=29740
for spec in C5:copy C2:copy C4:copy C5:inline C4:inline; do
  IFS=: read c mode <<< "$spec"
  port=$((port+1))
  BPC_NVLS_MODE=$mode timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --exchange nvls --steps 200 --warmup 10 --no-cpu --no-e2e > ${O}_bench_${c}_$mode.json 2> ${O}_bench_${c}_$mode.err
  echo "$c $mode rc=$?"
  tail -1 ${O}_bench_${c}_$mode.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['config']['exchange'], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})" 2>/dev/null
done
