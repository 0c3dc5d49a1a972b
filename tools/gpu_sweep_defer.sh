#!/bin/bash
# Emit-deferral sweep of the compression kernels (BPC_CSTREAM_DEFER = D): bench
# lines per D and config, after a parity pass at the default D.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py -x -q > gpurun_out/sw_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/sw_pytest.log
for D in 1 2 3; do
  for c in ${1:-C5 C2 C4 C3}; do
    BPC_CSTREAM_DEFER=$D timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/sw_${c}_D$D.json 2> gpurun_out/sw_${c}_D$D.err
    tail -1 gpurun_out/sw_${c}_D$D.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('D=$D', d['config']['workload'][:3], d['ms_per_step'], {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
  done
done
