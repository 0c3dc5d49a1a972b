#!/bin/bash
# driver-like pass: the whole -m gpu suite, smoke(), and the C3 timing-pass check
mkdir -p gpurun_out
O=gpurun_out/ck
start=$(date +%s)
timeout 2400 python -m pytest tests/ -x -q -m gpu > ${O}_pytest.log 2>&1; echo pytest=$? secs=$(( $(date +%s) - start )); tail -4 ${O}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo smoke=$?; tail -2 ${O}_smoke.log
for s in 200 1000; do
  timeout 300 python bench.py --config C3 --steps $s --warmup 10 --no-e2e --no-cpu > ${O}_C3_$s.json 2> ${O}_C3_$s.err
  tail -1 ${O}_C3_$s.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('steps $s', d['ms_per_step'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
done
