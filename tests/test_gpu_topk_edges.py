"""Top-k selection edge cases the synthetic gradients never produce (R9: order
by |q| descending then index ascending), against the oracle's
plain stable sort:
* an all-zero unit without error feedback (every key ties at 0: the histogram
  bin holding the k-th key overflows both 10-bit rounds -> the 4 x 8-bit
  cluster radix select, kernels_compress.cu's fallback);
* a constant unit (same);
* 300 entries tied at the k-th largest magnitude (the 257-512-candidate path
  after the refine round) and 600 tied entries (> 512: radix fallback with a
  tie cut in the middle of the tied run);
with and without EF, at n = 1 and over the product exchange at n = 2."""
import numpy as np
import pytest

from workloads import TOP_K, RANDOM_K, Comp, Config, layout

pytestmark = pytest.mark.gpu

SHAPES = (262144, 300000, 5000, 40000)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


def _grads(w, n, step):
    numels = w.tensor_numels()
    offs, D = layout(numels)
    rng = np.random.default_rng([11, step])
    gs = []
    for i in range(n):
        g = np.zeros(D, np.float32)
        if step == 1:
            pass                                          # all zero
        elif step == 2:
            g[:] = 0.0
            for o, L in zip(offs, numels):
                g[o:o + L] = np.float32(0.5 if i == 0 else -0.25)   # constant units
        else:
            for ti, (o, L) in enumerate(zip(offs, numels)):
                v = (rng.standard_normal(L) * 0.01).astype(np.float32)
                if ti == 0:        # 300 ties at the top magnitude of unit 0 (k = 262)
                    pos = rng.choice(L, 300, replace=False)
                    v[pos] = np.where(rng.random(300) < 0.5, 1.0, -1.0).astype(np.float32)
                if ti == 1:        # 600 ties in the first unit of tensor 1, 100 above them
                    pos = rng.choice(1 << 18, 700, replace=False)
                    v[pos[:600]] = np.float32(0.75)
                    v[pos[600:]] = np.float32(-2.0)
                g[o:o + L] = v
        gs.append(g)
    return gs


@pytest.mark.parametrize("mode,n", [("copy", 1), ("p2p", 2)])
@pytest.mark.parametrize("use_ef", [0, 1])
@pytest.mark.parametrize("kind", [TOP_K, RANDOM_K])
def test_sparse_ties_and_zeros(kind, use_ef, mode, n):
    import torch
    import oracle
    from gpu_harness import LoopbackGroup, compare_step, oracle_for
    w = Config("edges", "custom", Comp(kind, 1, 1000, use_ef=use_ef), numels=SHAPES, threshold_bytes=0)
    grp = LoopbackGroup(w, n, mode=mode)
    ocfg, ost = oracle_for(w, n)
    try:
        for step in (1, 2, 3, 4):
            gs = _grads(w, n, step)
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), 1e-3)
            grp.step([torch.tensor(g, device="cuda") for g in gs], 1e-3)
            compare_step(grp, ocfg, ost, delta, p, label=f"edges kind {kind} ef {use_ef} {mode} step {step}")
    finally:
        grp.close()
