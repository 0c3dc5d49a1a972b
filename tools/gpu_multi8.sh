# 8-GPU weak-scaling bench lines (fused NVLink exchange) + the 8-rank parity test
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/n8_gpus.txt 2>&1
for c in C2 C5 C3 C4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 8 --config $c --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_${c}_n8.log 2>&1
  echo "$c rc=$?" >> gpurun_out/n8_rc.txt
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "8-p2p or 8-nccl" > gpurun_out/multi8_pytest.log 2>&1; echo rc=$? >> gpurun_out/multi8_pytest.log
