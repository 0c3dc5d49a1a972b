#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/nv3
[ -x tools/nvls_bind_matrix ] || nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/nvls_bind_matrix tools/nvls_bind_matrix.cu -lcuda
timeout 120 ./tools/nvls_bind_matrix > ${O}_matrix.log 2>&1; cat ${O}_matrix.log
timeout 600 python -m pytest tests/test_gpu_nvls.py -x -q -rs > ${O}_nvls_pytest.log 2>&1; echo nvls_pytest=$?; tail -5 ${O}_nvls_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "2-nvls" > ${O}_multi_pytest.log 2>&1; echo multi_pytest=$?; tail -5 ${O}_multi_pytest.log
port=29690
for c in C5 C2; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --config $c --exchange nvls --steps 200 --warmup 10 --no-cpu --no-e2e > ${O}_bench_${c}_nvls.json 2> ${O}_bench_${c}_nvls.err
  echo "$c nvls rc=$?"
  tail -1 ${O}_bench_${c}_nvls.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['config']['exchange'], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})" 2>/dev/null
done
