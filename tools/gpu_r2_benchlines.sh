#!/bin/bash
# N = 1 bench lines with the full contract (after the summaries / traffic.json of
# tools/gpu_r2_final.sh are in profiles/r2), the default invocation and the reference arm
mkdir -p gpurun_out/bl
O=gpurun_out/bl
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
for c in C2 C3 C4 C5; do
  timeout 300 python bench.py --config $c > $O/bench_${c}_n1.json 2> $O/bench_${c}_n1.err; echo bench$c=$?
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
timeout 300 python bench.py --config C2 --launch eager > $O/bench_C2_n1_eager.json 2> $O/bench_C2_n1_eager.err; echo eager=$?
