#!/bin/bash
# One GPU-box pass over HEAD: smoke, the -m gpu suite, the default bench line,
# the reference arm, and the size-threshold search for C2 / C5.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 600 python tools/threshold_search.py --config C2 --steps 100 > gpurun_out/thr_C2.json 2> gpurun_out/thr_C2.err; echo thrC2=$?
timeout 900 python tools/threshold_search.py --config C5 --steps 30 > gpurun_out/thr_C5.json 2> gpurun_out/thr_C5.err; echo thrC5=$?
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_default.log
