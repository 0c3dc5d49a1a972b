#!/bin/bash
# Iteration pass: parity of the streaming kernels first (stop at the first
# failure), then bench lines, then (optional) ncu --set full of the named kernels.
# usage: tools/gpu_iter.sh "<pytest selection>" "<configs>" "<ncu config:regex:skip:count ...>"
mkdir -p gpurun_out
SEL=${1:-"tests/test_gpu_parity.py"}
if [ -n "$KSEL" ]; then timeout 1500 python -m pytest $SEL -k "$KSEL" -x -q > gpurun_out/iter_pytest.log 2>&1; else timeout 1500 python -m pytest $SEL -x -q > gpurun_out/iter_pytest.log 2>&1; fi; rc=$?; echo pytest=$rc
tail -15 gpurun_out/iter_pytest.log
[ $rc -ne 0 ] && exit 1
for c in ${2:-C5}; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/iter_bench_${c}.json 2> gpurun_out/iter_bench_${c}.err; echo bench$c=$?
  tail -1 gpurun_out/iter_bench_${c}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], d['ms_per_step'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
done
for spec in $3; do
  IFS=: read cfg kre skip cnt <<< "$spec"
  CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu"
  R=gpurun_out/iter_${cfg}_${kre}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c $cnt -o $R $CMD > gpurun_out/iter_ncu_${cfg}.log 2>&1; echo ncu$cfg=$?
  # keep the exports (small); the report itself only if KEEP_REP is set
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > ${R}_details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2>/dev/null
  gzip -f ${R}_sass.csv
  [ -z "$KEEP_REP" ] && rm -f $R.ncu-rep
done
du -sh gpurun_out
