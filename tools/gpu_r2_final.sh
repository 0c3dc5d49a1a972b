#!/bin/bash
# Round-2 evidence pass on ONE GPU (run on HEAD, results committed together):
#  1. bench lines with the full contract (roofline, cpu_baseline, e2e, clocks) for C2-C5
#     and the default invocation (C5);
#  2. the ncu launch list (gpu__time_duration + DRAM bytes) of the same bench command;
#  3. ncu --set full of one step's libbpc kernels, exported to CSV (raw page) for the
#     summaries and the roofline `traffic` (tools/r2_summarize.py).
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi -q -d CLOCK > $O/clocks.txt 2>&1
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
for c in C2 C3 C4 C5; do
  timeout 300 python bench.py --config $c > $O/bench_${c}_n1.json 2> $O/bench_${c}_n1.err; echo bench$c=$?
done
timeout 300 python bench.py --impl reference --config C5 --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref=$?
K='regex:cstream|update_stream|sparse|unit_tree|lans_coef|p2p'
for c in C2 C3 C4 C5; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" --csv --log-file $O/launches_${c}.csv $CMD > $O/launches_${c}.log 2>&1; echo launches$c=$?
  if [ $c = C3 ]; then S=33; N=11; else S=9; N=3; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s $S -c $N -o $O/full_${c} $CMD > $O/full_${c}.log 2>&1; echo full$c=$?
  ncu -i $O/full_${c}.ncu-rep --page raw --csv > $O/full_${c}_raw.csv 2>/dev/null
  rm -f $O/full_${c}.ncu-rep
done
du -sh $O
