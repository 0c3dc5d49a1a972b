CMD="python bench.py --config C5 --optimizer lans --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_lans.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active --clock-control none -k "regex:update|lans" -s 6 -c 6 --csv --log-file gpurun_out/lans_launches.csv $CMD > gpurun_out/ncu_lans.log 2>&1
