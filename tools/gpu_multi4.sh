cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi4_pytest.log 2>&1; echo rc=$? >> gpurun_out/multi4_pytest.log
for c in C2 C5 C3 C4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --config $c --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_${c}_n4_fin.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --config C5 --optimizer lans --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_C5_n4_lans.log 2>&1
