#!/bin/bash
# Round-2 baseline pass on HEAD: the -m gpu suite, C3/C4/C5 bench lines, and
# ncu --set full captures of the kernels round 2 works on (one ncu tool per command,
# each after its plain command exited 0).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_base.log 2>&1; echo pytest=$?
for c in C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_${c}_base.json 2> gpurun_out/bench_${c}_base.err; echo bench$c=$?
done
CMD="python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cstream_kernel -s 6 -c 2 -o gpurun_out/prof_C5_base $CMD > gpurun_out/ncu_C5.log 2>&1; echo ncuC5=$?
CMD="python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cstream_kernel -s 6 -c 2 -o gpurun_out/prof_C4_base $CMD > gpurun_out/ncu_C4.log 2>&1; echo ncuC4=$?
CMD="python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"compress_kernel" -s 6 -c 2 -o gpurun_out/prof_C3_base $CMD > gpurun_out/ncu_C3.log 2>&1; echo ncuC3=$?
tail -3 gpurun_out/pytest_gpu_base.log
