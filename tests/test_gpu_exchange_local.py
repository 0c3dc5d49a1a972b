"""The product exchange (A4 push, A8 pull; Alg. 4 l.6-12) on ONE
GPU: n contexts of this process wired by bpc_connect_local into one peer-memory
group, so the driver's single-GPU box runs exactly the kernels of the
multi-process P2P transport - the worker's fused stores into the owners' RECV
slots, the system-scope release / acquire epoch flags, the server's wait, the
update's bulk reads of p from the owner's P (norm-based kinds), and the copy +
flag-wait kernels of the sparse kinds.  Every payload (as received by its
owner), every p (in its owner's P), e, e~ bit-exact vs the oracle; m, v, x
within 1e-6 relative (bit-exact by construction)."""
import numpy as np
import pytest

from workloads import (LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config, config)

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("onebit_noef", Comp(SCALED_SIGN, use_ef=0)),
    ("topk_ef", Comp(TOP_K, 1, 1000, use_ef=1)),
    ("topk_f16_ef", Comp(TOP_K, 1, 1000, use_ef=1, f16=1)),
    ("randk_ef", Comp(RANDOM_K, 1, 32, use_ef=1)),
    ("randk_scaled", Comp(RANDOM_K, 1, 32, randk_scaled=1, use_ef=0)),
    ("ldither7", Comp(LINEAR_DITHER, bits=7, use_ef=0)),
    ("ldither2_ef", Comp(LINEAR_DITHER, bits=2, use_ef=1)),
    ("ndither3", Comp(NATURAL_DITHER, bits=3, use_ef=0)),
    ("none", Comp(NONE, use_ef=1)),
]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("name,comp", KINDS, ids=[k[0] for k in KINDS])
def test_p2p_local_parity(name, comp, n):
    from gpu_harness import run_parity
    w = Config("p2p", "custom", comp, numels=SHAPES)
    run_parity(w, n, steps=3, label=f"p2p {name} n={n}", mode="p2p")


@pytest.mark.parametrize("n", [2, 3, 8])
def test_p2p_local_onebit_more_ranks(n):
    from gpu_harness import run_parity
    w = Config("p2p", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES)
    run_parity(w, n, steps=2, label=f"p2p onebit n={n}", mode="p2p")


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("kind", ["onebit", "topk"])
def test_p2p_local_ranks_without_units(kind, n):
    # C1 (BASELINE.json configs[0]): d = 4096 is ONE unit, so n - 1 ranks own no
    # unit and their server only releases the pull flags (api.cu's n_sslices == 0
    # path / an empty copy job); 10 steps as the config states
    from gpu_harness import run_parity
    w = config("C1")
    if kind == "topk":
        w = config("C1", comp=Comp(TOP_K, 1, 1000, use_ef=1))
    run_parity(w, n, steps=10, label=f"C1 {kind} p2p n={n}", mode="p2p")


def test_p2p_local_back_to_back():
    # five steps issued without any host synchronisation: the epochs of
    # consecutive steps must not be confused (flags are monotonic per direction)
    import torch
    import oracle
    from gpu_harness import LoopbackGroup, compare_step, oracle_for
    from workloads import gen_grad
    for comp in (Comp(SCALED_SIGN, use_ef=1), Comp(TOP_K, 1, 1000, use_ef=1)):
        w = Config("p2p", "custom", comp, numels=SHAPES)
        n = 3
        grp = LoopbackGroup(w, n, mode="p2p")
        ocfg, ost = oracle_for(w, n)
        try:
            dg = {s: [torch.tensor(gen_grad(w, i, s), device="cuda") for i in range(n)] for s in range(1, 6)}
            torch.cuda.synchronize()
            for s in range(1, 6):
                delta, p, _ = oracle.round_(ocfg, ost, np.stack([gen_grad(w, i, s) for i in range(n)]), 1e-3)
                grp.step(dg[s], 1e-3, sync=False)
            for c in grp.ctxs:
                c.sync()
            compare_step(grp, ocfg, ost, delta, p, label=f"back-to-back kind {comp.kind} step 5")
        finally:
            grp.close()


@pytest.mark.parametrize("opt", ["lans", "nag"])
def test_p2p_local_optimizers(opt):
    from gpu_harness import run_parity
    for comp in (Comp(SCALED_SIGN, use_ef=1), Comp(TOP_K, 1, 1000, use_ef=1, f16=1)):
        w = Config("p2p", "custom", comp, numels=SHAPES, optimizer=opt, lr=1e-2 if opt == "lans" else 1e-3)
        run_parity(w, 2, steps=2, label=f"p2p {opt} kind {comp.kind}", mode="p2p")


def test_p2p_local_per_tensor_units():
    from gpu_harness import run_parity
    w = Config("p2p", "custom", Comp(SCALED_SIGN, use_ef=1), numels=(1000, 70000, 300000, 1500000, 5),
               chunk_elems=0)
    run_parity(w, 2, steps=2, label="p2p per-tensor units", mode="p2p")


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4])
def test_p2p_local_c5_quarter(n):
    # BERT-large at 1/4 of every tensor (n in {2, 4} on C5), the
    # product exchange, two steps
    from gpu_harness import run_parity
    w = config("C5", n=n, scale=4)
    run_parity(w, n, steps=2, label=f"C5/4 p2p n={n}", mode="p2p")


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_p2p_local_quarter(name):
    from gpu_harness import run_parity
    w = config(name, n=2, scale=4)
    run_parity(w, 2, steps=2, label=f"{name}/4 p2p n=2", mode="p2p")


def test_connect_local_rejects_bad_groups():
    import paper_2105_07829_b200 as bpc
    w = Config("p2p", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES)
    a = bpc.context_for(w, rank=0, world_size=2)
    b = bpc.context_for(w, rank=1, world_size=2)
    c = bpc.context_for(w, rank=0, world_size=1)
    try:
        with pytest.raises(bpc.BpcError):
            bpc.connect_local([b, a])          # rank order
        with pytest.raises(bpc.BpcError):
            bpc.connect_local([a, c])          # world size
        w2 = Config("p2p", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES[:3])
        d = bpc.context_for(w2, rank=1, world_size=2)
        with pytest.raises(bpc.BpcError):
            bpc.connect_local([a, d])          # plans differ
        d.finalize()
        bpc.connect_local([a, b])
        assert a.exchange == "p2p" and b.exchange == "p2p"
    finally:
        for x in (a, b, c):
            x.finalize()
