#!/bin/bash
# 2-GPU pass: NVLS multicast feasibility probe (tools/nvls_probe.cu), NCCL's NVLS
# detection, the multi-GPU parity tests and N=2 bench lines.
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/nv
[ -x tools/nvls_probe ] || nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
for mb in 4 64; do timeout 120 ./tools/nvls_probe $mb >> ${O}_probe.log 2>&1; echo "probe $mb rc=$?" >> ${O}_probe.log; done
cat ${O}_probe.log
cat > /tmp/ar.py <<'PY'
import os, torch, torch.distributed as dist
r = int(os.environ["RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
x = torch.ones(1 << 26, device="cuda")
for _ in range(3): dist.all_reduce(x)
torch.cuda.synchronize(); dist.destroy_process_group()
PY
NCCL_DEBUG=INFO timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 /tmp/ar.py > ${O}_nccl.log 2>&1
grep -i "nvls\|multicast" ${O}_nccl.log | head -5
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "2-" > ${O}_pytest.log 2>&1; echo pytest=$?; tail -3 ${O}_pytest.log
port=29650
for c in C5 C2 C4 C3; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --config $c --steps 200 --warmup 10 --no-cpu --no-e2e > ${O}_bench_$c.json 2> ${O}_bench_$c.err
  echo "$c rc=$?"
  tail -1 ${O}_bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})" 2>/dev/null
done
