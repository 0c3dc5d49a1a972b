"""CUDA path (libbpc.so through the C ABI) vs the CPU oracle, element by element.

Bit-exact: packed sign bits, scales, top-k / random-k indices and values,
dithering codes and norms, worker and server errors.  m, v, x: bit-exact by
construction (same IEEE op order); the bar in the test is the
north star's 1e-6 relative.  Sizes span several 2^14-element CTA slices,
several clusters and ragged tails; n > 1 ranks run on one GPU through the
loopback exchange (tests/gpu_harness.py).
"""
import pytest

from workloads import (LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config)

pytestmark = pytest.mark.gpu

# raw (1000, 70000 < 1 MiB), two compression units with a ragged tail (300000),
# an odd-length compressed tensor (262147), a tiny tensor (5)
SHAPES = (1000, 300000, 70000, 262147, 5)


def _cfg(comp, name="custom", shapes=SHAPES, **kw):
    return Config(name, "custom", comp, numels=tuple(shapes), **kw)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("onebit_noef", Comp(SCALED_SIGN, use_ef=0)),
    ("topk_ef", Comp(TOP_K, 1, 1000, use_ef=1)),
    ("topk_dense_ef", Comp(TOP_K, 1, 50, use_ef=1)),
    ("randk_ef", Comp(RANDOM_K, 1, 32, use_ef=1)),
    ("randk_scaled", Comp(RANDOM_K, 1, 32, randk_scaled=1, use_ef=0)),
    ("ldither7", Comp(LINEAR_DITHER, bits=7, use_ef=0)),
    ("ldither2_ef", Comp(LINEAR_DITHER, bits=2, use_ef=1)),
    ("ndither3", Comp(NATURAL_DITHER, bits=3, use_ef=0)),
    ("none", Comp(NONE, use_ef=1)),
    ("topk_f16_ef", Comp(TOP_K, 1, 1000, use_ef=1, f16=1)),          # R23: binary16 values
    ("randk_scaled_f16", Comp(RANDOM_K, 1, 32, randk_scaled=1, use_ef=0, f16=1)),
]


@pytest.mark.parametrize("name,comp", KINDS, ids=[k[0] for k in KINDS])
def test_parity_n1(name, comp):
    from gpu_harness import run_parity
    run_parity(_cfg(comp), 1, steps=3, label=name)


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("name,comp", KINDS, ids=[k[0] for k in KINDS])
def test_parity_loopback(name, comp, n):
    from gpu_harness import run_parity
    run_parity(_cfg(comp), n, steps=2, label=f"{name} n={n}")


@pytest.mark.parametrize("chunk", [1 << 14, 1 << 15, 1 << 17])
@pytest.mark.parametrize("name,comp", [KINDS[0], KINDS[2], KINDS[6]], ids=["onebit", "topk", "ldither"])
def test_parity_cluster_shapes(name, comp, chunk):
    from gpu_harness import run_parity
    run_parity(_cfg(comp, chunk_elems=chunk), 2, steps=2, label=f"{name} chunk={chunk}")


def test_c1_ten_steps():
    # BASELINE.json configs[0]: d=4096, 2 workers, onebit + EF, 10 steps
    from gpu_harness import run_parity
    from workloads import config
    run_parity(config("C1"), 2, steps=10, label="C1")


@pytest.mark.parametrize("name,comp", [KINDS[0], KINDS[2], KINDS[4], KINDS[6], KINDS[8]],
                         ids=["onebit", "topk", "randk", "ldither", "ndither"])
def test_edge_zeros_and_ties(name, comp):
    # ties variant (values on a 2^-10 sigma grid) and an all-zero gradient step
    import numpy as np
    import torch
    import oracle
    from gpu_harness import LoopbackGroup, compare_step, oracle_for
    from workloads import gen_grad
    w = _cfg(comp, ties=True, threshold_bytes=0, shapes=(4096, 40000, 7, 262144))
    grp = LoopbackGroup(w, 2)
    ocfg, ost = oracle_for(w, 2)
    try:
        for step in range(1, 4):
            gs = [gen_grad(w, i, step) for i in range(2)]
            if step == 2:
                gs = [np.zeros_like(g) for g in gs]
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), 1e-3)
            grp.step([torch.tensor(g, device="cuda") for g in gs], 1e-3)
            compare_step(grp, ocfg, ost, delta, p, label=f"{name} step {step}")
    finally:
        grp.close()
