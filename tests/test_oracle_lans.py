"""Pins of the oracle's LANS / CLAN block update (Alg. 5 lines 12-18,
PAPER.md:285-295; Alg. 2; reading R22), each against
something other than the oracle's own formula: the SPEC hand-evaluated step,
closed forms of special cases, the paper's update-norm bound, and Adam's
direction from torch.optim.Adam (a library routine)."""
import numpy as np
import pytest
import torch

import oracle

B1, B2, EPS = 0.9, 0.999, 1e-6


def f32(*a):
    return [np.ascontiguousarray(x, dtype=np.float32) for x in a]


def step(g, m, v, x, t, lr, wd=0.0, b1=B1, b2=B2, eps=EPS, al=0.01, au=10.0):
    oracle.lans_block(g, m, v, x, t, lr, b1, b2, eps, wd, al, au)


def test_spec_hand_step():
    # d=1, x=1, g=1, beta1=0.9, beta2=0.99, eps=1e-6, lambda=0,
    # phi = clamp[0.01, 10], eta=0.1: m~ = v~ = 1, both normalised terms = 1 -> x' = 0.9
    g, m, v, x = f32([1.0], [0.0], [0.0], [1.0])
    step(g, m, v, x, 1, 0.1, b1=0.9, b2=0.99)
    assert abs(float(x[0]) - 0.9) <= 1e-6


def test_zero_gradient_fixed_point():
    # g~ = 0, lambda = 0, fresh state -> both terms defined as 0 -> x unchanged
    rng = np.random.default_rng(1)
    x0 = rng.standard_normal(777).astype(np.float32)
    g, m, v = f32(np.zeros(777), np.zeros(777), np.zeros(777))
    x = x0.copy()
    step(g, m, v, x, 1, 0.1)
    assert x.tobytes() == x0.tobytes()


@pytest.mark.parametrize("scale", [1e-4, 0.3, 5.0, 300.0])   # ||x|| below, inside, above [alpha_l, alpha_u]
def test_first_step_moves_by_eta_phi(scale):
    # t = 1, m = v = 0, lambda = 0: m~ = g~, v~ = g~^2, so r = c and
    # d~ = phi(||x||) r/||r||: the block moves by exactly eta * clamp(||x||) (within fp32)
    rng = np.random.default_rng(2)
    n = 1000
    x0 = (rng.standard_normal(n) * scale / np.sqrt(n)).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    m, v = f32(np.zeros(n), np.zeros(n))
    x = x0.copy()
    lr = 1e-2
    step(g, m, v, x, 1, lr)
    phi = min(max(np.linalg.norm(x0.astype(np.float64)), 0.01), 10.0)
    moved = np.linalg.norm(x.astype(np.float64) - x0)
    # tolerance: the fp32 rounding of x' (half an ulp of |x| per coordinate, relative
    # to the per-coordinate move eta*phi/sqrt(n))
    rel = max(1e-5, 4 * 2.0 ** -24 * float(np.abs(x0).max()) * np.sqrt(n) / (lr * phi))
    assert moved == pytest.approx(lr * phi, rel=rel)
    # and along -sign(g): each coordinate moves against its gradient
    d = x.astype(np.float64) - x0
    nz = np.abs(d) > 0
    assert np.all(np.sign(d[nz]) == -np.sign(g[nz]))


def test_weight_decay_only_shrinks_along_x():
    # g~ = 0 forever, m = v = 0: r = c = 0, u = w = lambda x, d~ = phi(||x||) x/||x||
    # -> x' = x - eta phi x/||x|| (a dropped lambda or a sign error breaks it)
    rng = np.random.default_rng(3)
    n = 513
    x0 = rng.standard_normal(n).astype(np.float32)
    g, m, v = f32(np.zeros(n), np.zeros(n), np.zeros(n))
    x = x0.copy()
    lr = 0.05
    step(g, m, v, x, 1, lr, wd=0.01)
    x064 = x0.astype(np.float64)
    nx = np.linalg.norm(x064)
    want = x064 - lr * min(max(nx, 0.01), 10.0) * x064 / nx
    np.testing.assert_allclose(x, want, rtol=1e-6, atol=1e-7)


def test_update_norm_bound():
    # appendix Eq. (2): with lambda = 0 the block
    # moves by at most eta * phi(||x_b||) <= eta * alpha_u, every step
    rng = np.random.default_rng(4)
    n = 2048
    x = (rng.standard_normal(n) * 3).astype(np.float32)
    m, v = f32(np.zeros(n), np.zeros(n))
    lr = 0.1
    for t in range(1, 30):
        g = (rng.standard_normal(n) * 10 ** rng.uniform(-3, 1)).astype(np.float32)
        x0 = x.copy()
        step(g, m, v, x, t, lr)
        phi = min(max(np.linalg.norm(x0.astype(np.float64)), 0.01), 10.0)
        moved = np.linalg.norm(x.astype(np.float64) - x0)
        assert moved <= lr * phi * (1 + 1e-5) + 1e-9
        assert moved <= lr * 10.0 * (1 + 1e-5)


def test_momentum_term_against_torch_adam():
    # Coordinates whose current gradient is 0 have c = 0, so only the momentum
    # term moves them: dx_j = -eta phi beta1 r_j / ||r||, with r = Adam's step
    # direction (torch.optim.Adam, eps outside the sqrt).  Catches swapped
    # beta1 / (1 - beta1) or a wrong norm.
    rng = np.random.default_rng(5)
    n = 64
    g1 = rng.standard_normal(n).astype(np.float32)
    g2 = rng.standard_normal(n).astype(np.float32)
    g2[: n // 2] = 0.0
    x0 = rng.standard_normal(n).astype(np.float32)
    # torch Adam: r at t = 2 from the parameter change with lr = 1
    p = torch.nn.Parameter(torch.tensor(x0, dtype=torch.float64))
    opt = torch.optim.Adam([p], lr=1.0, betas=(B1, B2), eps=EPS)
    for g in (g1, g2):
        p.grad = torch.tensor(g, dtype=torch.float64)
        before = p.detach().clone()
        opt.step()
    r = (before - p.detach()).numpy()            # the t = 2 Adam direction m~/(sqrt(v~)+eps)
    # oracle LANS over the same two steps, lr = 0 at t = 1 so x stays x0
    m, v = f32(np.zeros(n), np.zeros(n))
    x = x0.copy()
    step(g1, m, v, x, 1, 0.0)
    lr = 1e-2
    step(g2, m, v, x, 2, lr)
    phi = min(max(np.linalg.norm(x0.astype(np.float64)), 0.01), 10.0)
    dx = x.astype(np.float64) - x0
    want = -lr * phi * B1 * r[: n // 2] / np.linalg.norm(r)
    np.testing.assert_allclose(dx[: n // 2], want, rtol=2e-4, atol=1e-9)


def test_round_lans_none_is_lans_of_the_mean():
    # Alg. 5 with the identity compressor (NONE) = LANS on push_pull(g)
    rng = np.random.default_rng(6)
    numels = [300, 5000, 17]
    offs = [0, 304, 5312]
    D = 5332
    comp = oracle_comp_none()
    cfg = oracle.Cfg(2, numels, offs, comp, threshold_bytes=0, optimizer="lans", weight_decay=0.01)
    x0 = rng.standard_normal(D).astype(np.float32)
    st = oracle.State(2, D, x0)
    grads = rng.standard_normal((2, D)).astype(np.float32)
    oracle.round_(cfg, st, grads, 1e-2, want_payloads=False)
    mean = oracle.push_pull(grads)
    for nl, o in zip(numels, offs):
        m, v = f32(np.zeros(nl), np.zeros(nl))
        x = x0[o:o + nl].copy()
        step(mean[o:o + nl], m, v, x, 1, 1e-2, wd=0.01)
        assert x.tobytes() == st.x[o:o + nl].tobytes()


def oracle_comp_none():
    from workloads import NONE, Comp
    return Comp(NONE, use_ef=0)
