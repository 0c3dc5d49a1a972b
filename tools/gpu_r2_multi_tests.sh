#!/bin/bash
# multi-GPU parity only (all transports, eager and graph) on N GPUs
N=${1:-4}
mkdir -p gpurun_out/scale
timeout 2000 python -m pytest tests/test_gpu_multi.py tests/test_gpu_nvls.py -q -rs -k "$N- or nvls_local" > gpurun_out/scale/n${N}_pytest_full.log 2>&1; echo pytest=$?; tail -4 gpurun_out/scale/n${N}_pytest_full.log
