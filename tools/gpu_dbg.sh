mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "randk_ef-3 or randk_ef-4 or randk_scaled-3" > gpurun_out/dbg.log 2>&1; echo rc=$?
grep -E "Error|error|bpc_|Mismatch|passed|failed" gpurun_out/dbg.log | head -30
