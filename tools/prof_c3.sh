CMD="python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_C3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress_kernel" -s 2 -c 2 -o gpurun_out/prof_C3_topk $CMD > gpurun_out/ncu_C3.log 2>&1
echo done
