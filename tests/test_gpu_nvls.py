"""The NVLS multicast pull (`PAPER.md:491-492`; include/bpc.h
BPC_EXCHANGE_NVLS) on one process over n distinct GPUs (bpc_connect_local):
the server kernel stores p once through the multicast mapping of P and the
switch writes it into every rank's P; the update reads it locally.  Every
rank's P must then hold every unit's p (bit-exact vs the oracle), with e, e~
bit-exact and m, v, x within 1e-6.  Skips on a box with one GPU or without
multicast support (the multi-process path: tests/test_gpu_multi.py nvls)."""
import numpy as np
import pytest

from workloads import LINEAR_DITHER, NONE, SCALED_SIGN, Comp, Config, gen_grad, gen_params

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5, 600000)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("ldither7", Comp(LINEAR_DITHER, bits=7, use_ef=0)),
    ("none", Comp(NONE, use_ef=1)),
]


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


class NvlsGroup:
    def __init__(self, w, n):
        import torch
        import paper_2105_07829_b200 as bpc
        self.w, self.n, self.fused = w, n, True
        self.ctxs = []
        for r in range(n):
            with torch.cuda.device(r):
                self.ctxs.append(bpc.context_for(w, rank=r, world_size=n, device=r, check_finite=1,
                                                 exchange="nvls"))
        bpc.connect_local(self.ctxs)
        self.x = [torch.tensor(gen_params(w), device=f"cuda:{r}") for r in range(n)]

    def step(self, grads, lr):
        for i, c in enumerate(self.ctxs):
            c.compress(grads[i])
        for c in self.ctxs:
            c.exchange_push()
        for c in self.ctxs:
            c.server()
        for c in self.ctxs:
            c.exchange_pull()
        for i, c in enumerate(self.ctxs):
            c.step(self.x[i], lr)
        for c in self.ctxs:
            c.sync()

    def close(self):
        for c in self.ctxs:
            c.finalize()


@pytest.mark.parametrize("name,comp", KINDS, ids=[k[0] for k in KINDS])
def test_nvls_local_group(name, comp):
    n = min(_ngpus(), 4)
    if n < 2:
        pytest.skip("needs 2 GPUs")
    import torch
    import oracle
    import paper_2105_07829_b200 as bpc
    from gpu_harness import compare_step, oracle_for
    w = Config("nvls", "custom", comp, numels=SHAPES)
    grp = NvlsGroup(w, n)
    try:
        if grp.ctxs[0].exchange != "nvls":
            pytest.skip("no NVLS multicast on this box: " + (bpc.lib().bpc_last_error(grp.ctxs[0].h) or b"").decode())
        ocfg, ost = oracle_for(w, n)
        lay = ocfg.payload_layout()
        for step in range(1, 4):
            gs = [gen_grad(w, i, step) for i in range(n)]
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), 1e-3)
            grp.step([torch.tensor(gs[i], device=f"cuda:{i}") for i in range(n)], 1e-3)
            compare_step(grp, ocfg, ost, delta, p, label=f"nvls {name} step {step}")
            # every rank's P holds every unit's p (the multicast reached all replicas)
            for i, c in enumerate(grp.ctxs):
                pb = c.copy_state(bpc.BUF_P)
                for ci, gc in enumerate(c.chunks()):
                    po, nb = lay[ci]
                    assert pb[gc.payload_offset:gc.payload_offset + nb].tobytes() == p[po:po + nb].tobytes(), \
                        f"rank {i}: p of chunk {ci} (owner {gc.owner}) missing from its P"
    finally:
        grp.close()
