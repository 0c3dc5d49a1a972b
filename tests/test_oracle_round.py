"""Pins for the oracle's whole round (Alg. 3/4 + Alg. 5 lines 12-18).

Hand traces of Alg. 4 (golden files), SPEC's Alg. 4 trace, identity
recovery of Alg. 1, the EF reconstruction identities
(PAPER.md:245, 257), Adam against torch.optim (a library routine), the
Lemma-2 residual bounds and the chunk plan.
"""
import json
import math
import os
import struct

import numpy as np
import pytest

from workloads import (LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp,
                       config, gen_grad, gen_params, layout)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _cfg(orc, n, numels, comp, **kw):
    offs, D = layout(numels)
    kw.setdefault("threshold_bytes", 0)
    return orc.Cfg(n, numels, offs, comp, **kw), D


def test_onebit_two_worker_trace(orc):
    gold = json.load(open(os.path.join(GOLDEN, "onebit_ef_trace.json")))
    cfg, D = _cfg(orc, 2, [4], Comp(SCALED_SIGN, use_ef=1))
    st = orc.State(2, D, np.zeros(D, np.float32))
    g = np.zeros((2, D), np.float32)
    g[:, :4] = gold["g"]
    for step in gold["steps"]:
        etilde_before = st.et[:4].copy()
        delta, p, gt = orc.round_(cfg, st, g, lr=0.0)
        for i in range(2):
            s, bits = struct.unpack("<fB", delta[i, :5].tobytes())
            assert s == step["s"][i] and bits == step["bits"][i]
            assert list(st.e[i, :4]) == step["e"][i]
        s_p, bits_p = struct.unpack("<fB", p[:5].tobytes())
        assert s_p == step["s_p"] and bits_p == step["bits_p"]
        assert list(st.et[:4]) == step["etilde"]
        # Delta = dec(p) + e~_{t+1} exactly (Alg. 4 line 13, every value exact here)
        assert list(gt[:4] + st.et[:4]) == step["Delta"]
        del etilde_before


def test_topk_two_worker_trace_with_ties(orc):
    gold = json.load(open(os.path.join(GOLDEN, "topk_ef_trace.json")))
    cfg, D = _cfg(orc, 2, [4], Comp(TOP_K, k_num=1, k_den=4, use_ef=1))
    st = orc.State(2, D, np.zeros(D, np.float32))
    g = np.zeros((2, D), np.float32)
    g[:, :4] = gold["g"]
    for step in gold["steps"]:
        delta, p, gt = orc.round_(cfg, st, g, lr=0.0)
        for i in range(2):
            k, idx = struct.unpack("<QI", delta[i, :12].tobytes())
            assert k == 1 and idx == step["idx"][i]
            assert list(st.e[i, :4]) == step["e"][i]
        k, idx, val = struct.unpack("<QIf", p[:16].tobytes())
        assert (idx, val) == (step["p_idx"], step["p_val"])
        assert list(st.et[:4]) == step["etilde"]


def test_spec_alg4_hand_trace(orc):
    # n=1, top-k k=1, g=[3,1] -> output [3,0]; then g=[0,2] -> [0,3]
    cfg, D = _cfg(orc, 1, [2], Comp(TOP_K, k_num=1, k_den=2, use_ef=1))
    st = orc.State(1, D, np.zeros(D, np.float32))
    g = np.zeros((1, D), np.float32)
    g[0, :2] = [3, 1]
    _, _, gt = orc.round_(cfg, st, g, 0.0)
    assert list(gt[:2]) == [3, 0] and list(st.e[0, :2]) == [0, 1]
    g[0, :2] = [0, 2]
    _, _, gt = orc.round_(cfg, st, g, 0.0)
    assert list(gt[:2]) == [0, 3] and list(st.e[0, :2]) == [0, 0]


def test_spec_alg3_onebit_two_way(orc):
    # n=1, scaled sign, g=[1,-2,3] -> worker sends [2,-2,2], server
    # re-compresses to [2,-2,2]
    cfg, D = _cfg(orc, 1, [3], Comp(SCALED_SIGN, use_ef=0))
    st = orc.State(1, D, np.zeros(D, np.float32))
    g = np.zeros((1, D), np.float32)
    g[0, :3] = [1, -2, 3]
    _, _, gt = orc.round_(cfg, st, g, 0.0)
    assert list(gt[:3]) == [2, -2, 2]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("use_ef", [0, 1])
def test_identity_compressor_recovers_push_pull(orc, n, use_ef):
    # "When C is an identity mapping, both Algorithms ... recover
    # Algorithm 1". p_t = (1/n) sum g_i: compare with the exactly rounded mean.
    numels = [1000, 37, 5000]
    cfg, D = _cfg(orc, n, numels, Comp(NONE, use_ef=use_ef))
    rng = np.random.default_rng(n)
    g = rng.standard_normal((n, D)).astype(np.float32)
    st = orc.State(n, D, np.zeros(D, np.float32))
    _, _, gt = orc.round_(cfg, st, g, 0.0)
    pp = orc.push_pull(g)
    offs, _ = layout(numels)
    for o, L in zip(offs, numels):
        assert np.array_equal(gt[o:o + L], pp[o:o + L])
        exact = np.array([math.fsum(g[:, j].astype(np.float64)) / n for j in range(o, o + L)])
        assert np.all(np.abs(gt[o:o + L] - exact) <= np.spacing(np.abs(exact).astype(np.float32)) * 0.5 + 1e-45)
    assert not st.e.any() and not st.et.any()


@pytest.mark.parametrize("kind", [SCALED_SIGN, TOP_K, RANDOM_K, LINEAR_DITHER, NATURAL_DITHER])
def test_ef_reconstruction_identities(orc, kind):
    # Alg. 4 lines 7 and 13: e' = q - dec(delta) and
    # e~' = Delta - dec(p) as binary32 operations (R18); exact for sparse kinds.
    numels = [3000, 700]
    comp = Comp(kind, k_num=1, k_den=50, bits=5, use_ef=1)
    cfg, D = _cfg(orc, 2, numels, comp, chunk_elems=1024, seed=17)
    rng = np.random.default_rng(kind)
    st = orc.State(2, D, np.zeros(D, np.float32))
    for step in range(3):
        g = rng.standard_normal((2, D)).astype(np.float32)
        e_before = st.e.copy()
        et_before = st.et.copy()
        delta, p, gt = orc.round_(cfg, st, g, 0.0)
        lay = cfg.payload_layout()
        for ci, (ti, off, L, raw) in enumerate(cfg.plan()):
            po, pb = lay[ci]
            dsum = np.zeros(L)
            for i in range(2):
                q = g[i, off:off + L] + e_before[i, off:off + L]
                dec = orc.decompress(comp, delta[i, po:po + pb].tobytes(), L)
                assert np.array_equal(st.e[i, off:off + L], q - dec)
                if kind in (TOP_K, RANDOM_K):
                    assert np.array_equal(dec + st.e[i, off:off + L], q)
                dsum += dec.astype(np.float64)
            Delta = (dsum * 0.5 + et_before[off:off + L].astype(np.float64)).astype(np.float32)
            assert np.array_equal(st.et[off:off + L], Delta - gt[off:off + L])


@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_adam_matches_torch(orc, wd):
    # n=1 + NONE => Alg. 5 lines 12-18 reduce to Adam/AdamW; torch.optim is the
    # independent library routine (tolerance 1e-6 of the operands, R15).
    import torch
    rng = np.random.default_rng(0)
    D = 2048
    x0 = (rng.standard_normal(D) * 0.02).astype(np.float32)
    cfg, Dp = _cfg(orc, 1, [D], Comp(NONE), beta1=0.9, beta2=0.999, eps=1e-6, weight_decay=wd)
    st = orc.State(1, Dp, np.zeros(Dp, np.float32))
    st.x[:D] = x0
    xt = torch.tensor(x0.astype(np.float64), requires_grad=True)
    opt = (torch.optim.AdamW if wd else torch.optim.Adam)([xt], lr=1e-3, betas=(0.9, 0.999), eps=1e-6,
                                                          weight_decay=wd, foreach=False)
    for step in range(10):
        g = np.zeros((1, Dp), np.float32)
        g[0, :D] = (rng.standard_normal(D) * 10.0 ** rng.uniform(-4, -1)).astype(np.float32)
        orc.round_(cfg, st, g, 1e-3)
        xt.grad = torch.tensor(g[0, :D].astype(np.float64))
        opt.step()
        ref = xt.detach().numpy()
        assert np.all(np.abs(st.x[:D] - ref) <= 1e-6 * (np.abs(ref) + 1e-3))
    assert st.t == 11


def test_adam_first_step_bias_correction(orc):
    # at t=1, m~ = g~ and v~ = g~^2 in R (bias correction, Alg. 5
    # l.14-15), so with eps = 0, lambda = 0, lr = 1 and x = 0 the
    # step is x = -r = -g/|g| = -sign(g).  In fp32 m~ = fl(fl((1-b1) g)/(1-b1)) is
    # within 1 ulp of g (not always equal: DESIGN.md R16), v~ within 2 ulp of g^2,
    # so r is within a few ulp of +-1 (bound 8 ulp(1)).  A dropped bias correction
    # (r = 0.1 g / sqrt(0.001 g^2) = 3.16 sign(g)) or a swapped beta fails it.
    D = 64
    g = np.linspace(-1, 1, D).astype(np.float32)
    g = g[g != 0]
    m = np.zeros(g.size, np.float32)
    v = np.zeros(g.size, np.float32)
    x = np.zeros(g.size, np.float32)
    orc.adam(g, m, v, x, 1, 1.0, 0.9, 0.999, 0.0, 0.0)
    assert np.all(np.abs(-x - np.sign(g)) <= 8 * np.spacing(np.float32(1)))
    # second step, g repeated: m~ = g and v~ = g^2 again in R (both moments are
    # bias-corrected averages of identical terms), so x moves by -sign(g) again
    orc.adam(g, m, v, x, 2, 1.0, 0.9, 0.999, 0.0, 0.0)
    assert np.all(np.abs(-x - 2 * np.sign(g)) <= 16 * np.spacing(np.float32(1)))


@pytest.mark.parametrize("kind", [SCALED_SIGN, TOP_K])
def test_lemma2_residual_bounds(orc, kind):
    # PAPER.md:1123-1164 (Lemma 2): ||e_{t,i}|| <= sqrt(d(1-delta))/(1-sqrt(1-delta)) G;
    # with the delta each compressor certifies (top-k -> k/d).
    d = 64
    k_den = 8
    comp = Comp(kind, k_num=1, k_den=k_den, use_ef=1)
    cfg, D = _cfg(orc, 2, [d], comp)
    rng = np.random.default_rng(9)
    st = orc.State(2, D, np.zeros(D, np.float32))
    G = 1.0
    delta = 1.0 / k_den if kind == TOP_K else None
    for t in range(60):
        g = np.zeros((2, D), np.float32)
        g[:, :d] = rng.uniform(-G, G, size=(2, d)).astype(np.float32)
        if kind == SCALED_SIGN:
            # scaled sign certifies delta = ||q||_1^2 / (d ||q||^2) >= 1/d
            delta = 1.0 / d
        orc.round_(cfg, st, g, 0.0)
        a = math.sqrt(1 - delta)
        wb = math.sqrt(d * (1 - delta)) / (1 - a) * G
        sb = 2 * a / (1 - a) * (1 + wb / G) * G * math.sqrt(d)
        for i in range(2):
            assert np.linalg.norm(st.e[i, :d]) <= wb * (1 + 1e-6)
        assert np.linalg.norm(st.et[:d]) <= sb * (1 + 1e-6)


def test_chunk_plan(orc):
    # R1/R3: tensors with 4*numel < threshold stay raw (one unit); others split
    numels = [100, 262144, 262145, 700000, 5]
    offs, D = layout(numels)
    cfg = orc.Cfg(2, numels, offs, Comp(SCALED_SIGN), threshold_bytes=1 << 20, chunk_elems=1 << 18)
    plan = cfg.plan()
    assert [(t, L, r) for (t, _, L, r) in plan] == [
        (0, 100, 1), (1, 262144, 0), (2, 262144, 0), (2, 1, 0),
        (3, 262144, 0), (3, 262144, 0), (3, 175712, 0), (4, 5, 1)]
    covered = np.zeros(D, bool)
    for (t, o, L, r) in plan:
        assert not covered[o:o + L].any()
        covered[o:o + L] = True
    for o, L in zip(offs, numels):
        assert covered[o:o + L].all()
    # per-tensor units (R1 paper-faithful variant) and threshold 0
    cfg0 = orc.Cfg(2, numels, offs, Comp(SCALED_SIGN), threshold_bytes=0, chunk_elems=0)
    assert [(t, L, r) for (t, _, L, r) in cfg0.plan()] == [(i, L, 0) for i, L in enumerate(numels)]


def test_round_deterministic_and_c1_fast(orc):
    import time
    w = config("C1")
    cfg = orc.Cfg.from_workload(w)
    offs, D = layout(w.tensor_numels())
    runs = []
    t0 = time.time()
    for rep in range(2):
        st = orc.State(w.n, D, gen_params(w))
        for step in range(1, w.steps + 1):
            g = np.stack([gen_grad(w, i, step) for i in range(w.n)])
            orc.round_(cfg, st, g, w.lr)
        runs.append((st.x.copy(), st.e.copy(), st.et.copy(), st.m.copy(), st.v.copy()))
    assert time.time() - t0 < 10.0   # "CPU oracle in seconds" (BASELINE.json configs[0])
    for a, b in zip(*runs):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_round_thread_count_invariant(orc, name):
    # the OpenMP build (bench.py's all-cores cpu_baseline) must give the serial
    # result bit for bit: units are independent in Alg. 3/4 and the update
    w = config(name, n=2, scale=64)
    cfg = orc.Cfg.from_workload(w)
    offs, D = layout(w.tensor_numels())
    outs = []
    for threads in (1, 4):
        orc.set_threads(threads)
        st = orc.State(w.n, D, gen_params(w))
        for step in (1, 2):
            g = np.stack([gen_grad(w, i, step) for i in range(w.n)])
            d, p, _ = orc.round_(cfg, st, g, w.lr)
        outs.append((d.tobytes(), p.tobytes(), st.e.tobytes(), st.et.tobytes(), st.m.tobytes(), st.x.tobytes()))
    orc.set_threads(1)
    assert outs[0] == outs[1]
