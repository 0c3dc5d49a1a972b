#!/bin/bash
# Round-2 multi-GPU pass on one box of N GPUs: parity through both transports
# (eager and CUDA-graph replay), weak-scaling bench lines C2-C5 (graph replay,
# fused exchange), the C5 NCCL bus-bandwidth line, and the NVLink byte counters
# of the fused kernels (in-process group under ncu).
# usage: tools/gpu_r2_multi.sh N
N=${1:-2}
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
O=gpurun_out/r2m_n$N
nvidia-smi -L > ${O}_gpus.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > ${O}_pytest.log 2>&1; echo pytest=$? | tee -a ${O}_rc.txt
tail -5 ${O}_pytest.log
port=29611
run() {  # name, args...
  local name=$1; shift
  port=$((port+1))
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus $N "$@" > ${O}_bench_${name}.json 2> ${O}_bench_${name}.err
  echo "$name rc=$?" | tee -a ${O}_rc.txt
  tail -1 ${O}_bench_${name}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['ms_per_step'], d['value'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d.get('bus'))" 2>/dev/null
}
for c in C2 C5 C3 C4; do run $c --config $c --steps 200 --warmup 10 --no-cpu --no-e2e; done
run C5_nccl --config C5 --exchange nccl --steps 100 --warmup 10 --no-cpu --no-e2e
run C3_nccl --config C3 --exchange nccl --steps 100 --warmup 10 --no-cpu --no-e2e
run C2_eager --config C2 --launch eager --steps 200 --warmup 10 --no-cpu --no-e2e
run C5_e2e --config C5 --steps 50 --warmup 5 --no-cpu
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in C5 C2 C3; do
  timeout 600 ncu --metrics $M -k regex:"cstream|update|p2p|sparse" --clock-control none --csv --log-file ${O}_nvlink_${c}.csv python tools/nvlink_probe.py --config $c --n 2 --steps 2 > ${O}_nvlink_${c}.log 2>&1
  echo "nvlink $c rc=$?" | tee -a ${O}_rc.txt
done
timeout 300 python tools/nvlink_probe.py --config C5 --n $N --steps 3 > ${O}_probe_C5.log 2>&1; echo "probe rc=$?" | tee -a ${O}_rc.txt
