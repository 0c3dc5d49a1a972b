#!/bin/bash
# Round-2 check pass: the new exchange / edge tests first (bounded), the whole
# -m gpu suite, smoke, then the default bench line (C5, N=1) and C2/C3/C4 lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exchange_local.py tests/test_gpu_topk_edges.py -x -q > gpurun_out/pytest_new.log 2>&1; echo new=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
for c in C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 200 --no-e2e --no-cpu > gpurun_out/bench_${c}.json 2> gpurun_out/bench_${c}.err; echo bench$c=$?
done
tail -3 gpurun_out/pytest_new.log; tail -3 gpurun_out/pytest_gpu.log
