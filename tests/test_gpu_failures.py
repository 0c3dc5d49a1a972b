"""Failure detection through the C ABI: a non-finite gradient is
flagged by the worker kernels and reported by bpc_sync as BPC_ERR_NONFINITE
(status 7), for streaming, cluster (top-k) and raw units; the flag clears.
Host-detectable misuse (call order) is rejected before anything is enqueued."""
import numpy as np
import pytest
import torch

from workloads import LINEAR_DITHER, SCALED_SIGN, TOP_K, Comp, Config, gen_grad, gen_params

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


@pytest.mark.parametrize("where", [10, 1000 + 5, 1000 + 300000 + 7])   # raw, compressed, raw tensor
@pytest.mark.parametrize("comp", [Comp(SCALED_SIGN, use_ef=1), Comp(TOP_K, 1, 1000, use_ef=1),
                                  Comp(LINEAR_DITHER, bits=7, use_ef=0)], ids=["onebit", "topk", "ldither"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_nonfinite_gradient_is_reported(comp, where, bad):
    import paper_2105_07829_b200 as bpc
    from workloads import layout
    w = Config("fail", "custom", comp, numels=SHAPES)
    offs, D = layout(w.tensor_numels())
    ctx = bpc.context_for(w, check_finite=1)
    x = torch.tensor(gen_params(w), device="cuda")
    g = gen_grad(w, 0, 1)
    # flat index of element `where` of the concatenated tensors
    idx, acc = None, 0
    for o, n in zip(offs, SHAPES):
        if where < acc + n:
            idx = o + (where - acc)
            break
        acc += n
    g[idx] = bad
    ctx.compress(torch.tensor(g, device="cuda"))
    ctx.aggregate()
    ctx.step(x, w.lr)
    with pytest.raises(bpc.BpcError) as ei:
        ctx.sync()
    assert ei.value.status == 7
    # the flag clears: a clean step syncs
    ctx.compress(torch.tensor(gen_grad(w, 0, 2), device="cuda"))
    ctx.aggregate()
    ctx.step(x, w.lr)
    ctx.sync()
    ctx.finalize()


def test_call_order_is_enforced():
    import paper_2105_07829_b200 as bpc
    w = Config("fail", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES)
    ctx = bpc.context_for(w)
    x = torch.tensor(gen_params(w), device="cuda")
    with pytest.raises(bpc.BpcError) as ei:
        ctx.step(x, w.lr)                 # step before compress / aggregate
    assert ei.value.status == 6
    with pytest.raises(bpc.BpcError):
        ctx.aggregate()                   # aggregate before compress
    ctx.compress(torch.tensor(gen_grad(w, 0, 1), device="cuda"))
    with pytest.raises(bpc.BpcError):
        ctx.compress(torch.tensor(gen_grad(w, 0, 1), device="cuda"))   # twice
    ctx.aggregate()
    ctx.step(x, w.lr)
    ctx.sync()
    ctx.finalize()
