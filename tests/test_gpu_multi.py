"""Multi-GPU parity through the NVLink peer-store exchange and NCCL (bpc_aggregate): torchrun one process per GPU
on 2 (and 4, 8 when present) B200s; every rank's payloads, errors and parameters
are checked against the CPU oracle (tests/multigpu_parity.py).  Skips when the
box has a single GPU (the loopback tests cover n > 1 there)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("launch", ["eager", "graph"])
@pytest.mark.parametrize("exchange", ["p2p", "nccl", "nvls"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_parity(n, exchange, launch):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    import socket
    for attempt in range(3):   # the rendezvous port can be taken between the probe and the bind
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.join(ROOT, "tests", "multigpu_parity.py"), "", exchange, launch]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        out = r.stdout + r.stderr
        if r.returncode == 0 or "EADDRINUSE" not in out:
            break
    assert r.returncode == 0, out[-4000:]
    for rank in range(n):
        for name in ("onebit", "topk", "randk", "ldither", "lans_onebit", "lans_topk", "units_onebit", "nag_topk"):
            assert f"RANK {rank} {name} OK" in out, out[-4000:]
