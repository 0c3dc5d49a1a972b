"""Checkpoint / resume through the C ABI (bpc_copy_state, bpc_load_state,
bpc_set_step): 2 steps, save e, e~, m, v, t and x, rebuild the context, load,
2 more steps == 4 uninterrupted steps, bit for bit (SURVEY.md aux subsystem)."""
import numpy as np
import pytest
import torch

from workloads import SCALED_SIGN, TOP_K, Comp, Config, gen_grad, gen_params

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5)
BUFS = None


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


def _run(ctx, x, w, steps):
    for step in steps:
        g = torch.tensor(gen_grad(w, 0, step), device="cuda")
        ctx.compress(g)
        ctx.aggregate()
        ctx.step(x, w.lr)
    ctx.sync()


@pytest.mark.parametrize("name,comp,opt", [
    ("onebit_adam", Comp(SCALED_SIGN, use_ef=1), "adam"),
    ("topk_lans", Comp(TOP_K, 1, 1000, use_ef=1, f16=1), "lans"),
    ("onebit_nag", Comp(SCALED_SIGN, use_ef=1), "nag"),
])
def test_resume_is_bit_exact(name, comp, opt):
    import paper_2105_07829_b200 as bpc
    bufs = [bpc.BUF_WORKER_ERR, bpc.BUF_SERVER_ERR, bpc.BUF_M, bpc.BUF_V]
    w = Config("ckpt", "custom", comp, numels=SHAPES, optimizer=opt, lr=1e-2)
    # uninterrupted
    a = bpc.context_for(w)
    xa = torch.tensor(gen_params(w), device="cuda")
    _run(a, xa, w, [1, 2, 3, 4])
    want = {b: a.copy_state(b) for b in bufs}
    a.finalize()
    # interrupted after 2 steps
    b1 = bpc.context_for(w)
    xb = torch.tensor(gen_params(w), device="cuda")
    _run(b1, xb, w, [1, 2])
    saved = {b: b1.copy_state(b) for b in bufs}
    t = b1.t
    x_host = xb.cpu().numpy().copy()
    b1.finalize()
    b2 = bpc.context_for(w)
    for b, data in saved.items():
        b2.load_state(b, data)
    b2.set_step(t)
    xb2 = torch.tensor(x_host, device="cuda")
    _run(b2, xb2, w, [3, 4])
    assert b2.t == 5
    assert xb2.cpu().numpy().tobytes() == xa.cpu().numpy().tobytes()
    for b in bufs:
        assert np.array_equal(b2.copy_state(b), want[b]), f"{name}: buffer {b} differs after resume"
    b2.finalize()
