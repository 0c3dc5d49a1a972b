"""Pins for the oracle's compression operators.

Each check is fixed by the paper or by mathematics, not by the oracle:
SPEC's worked examples (derived from the paper's definitions), the sign(0)
example, the scaled-sign error closed form, brute-force characterisation of
top-k, enumerations and Monte-Carlo unbiasedness (Def. 1),
and the closed-form payload sizes.
"""
import itertools
import struct

import numpy as np
import pytest

from workloads import LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K


def C(orc, kind, **kw):
    return orc.comp_struct(kind, **kw)


# ---------------------------------------------------------------- onebit
def test_onebit_spec_example(orc):
    # [1,-2,3] -> scale ||x||_1/d = 2, signs (+,-,+)
    p = orc.compress(C(orc, SCALED_SIGN), [1, -2, 3])
    assert p == bytes.fromhex("0000004005")
    assert list(orc.decompress(C(orc, SCALED_SIGN), p, 3)) == [2, -2, 2]


def test_onebit_sign_of_zero(orc):
    # x=[1,0,0,0] -> ||C(x)-x||^2 = 3/16 + (3/4)^2 = 0.75; holds only
    # with sign(0) = +1 (R2), also for -0.
    for x in ([1, 0, 0, 0], [1, -0.0, 0, -0.0]):
        p = orc.compress(C(orc, SCALED_SIGN), x)
        assert p[4] == 0x0F
        d = orc.decompress(C(orc, SCALED_SIGN), p, 4)
        assert float(np.sum((d - np.float32(x)) ** 2)) == 0.75


def test_onebit_error_closed_form(orc):
    # ||C(x)-x||^2 = ||x||^2 - ||x||_1^2 / d for C(x) = ||x||_1/d sign(x) (in R);
    # this is also Def. 2 with delta = ||x||_1^2 / (d ||x||^2).
    rng = np.random.default_rng(1)
    for d in (1, 2, 5, 31, 32, 33, 1000, 4099):
        x = (rng.standard_normal(d) * 10.0 ** rng.uniform(-3, 1)).astype(np.float32)
        dec = orc.decompress(C(orc, SCALED_SIGN), orc.compress(C(orc, SCALED_SIGN), x), d).astype(np.float64)
        xd = x.astype(np.float64)
        lhs = np.sum((dec - xd) ** 2)
        rhs = np.sum(xd ** 2) - np.sum(np.abs(xd)) ** 2 / d
        assert abs(lhs - rhs) <= 1e-5 * np.sum(xd ** 2) + 1e-30
        assert lhs <= (1 - np.sum(np.abs(xd)) ** 2 / (d * np.sum(xd ** 2))) * np.sum(xd ** 2) * (1 + 1e-5) + 1e-30


def test_onebit_payload_layout(orc):
    # bit j of byte j>>3 at position j&7, 1 = nonnegative
    x = np.array([(-1.0) ** (j * j // 3) * (j + 1) for j in range(19)], dtype=np.float32)
    p = orc.compress(C(orc, SCALED_SIGN), x)
    assert len(p) == 4 + 3
    s = struct.unpack("<f", p[:4])[0]
    assert s == np.float32(np.sum(np.abs(x.astype(np.float64))) / 19)
    for j in range(19):
        assert ((p[4 + (j >> 3)] >> (j & 7)) & 1) == (1 if x[j] >= 0 else 0)
    assert p[6] >> 3 == 0  # unused tail bits are 0


def test_onebit_compression_rate(orc):
    # d = 10^6 -> 4e6 / (1e6/8 + 4) = 31.999
    assert abs(4e6 / orc.payload_bytes(C(orc, SCALED_SIGN), 0, 10 ** 6) - 31.999) < 1e-3


# ---------------------------------------------------------------- top-k
def _sparse(p):
    k = struct.unpack("<Q", p[:8])[0]
    idx = list(struct.unpack(f"<{k}I", p[8:8 + 4 * k]))
    val = list(struct.unpack(f"<{k}f", p[8 + 4 * k:8 + 8 * k]))
    return k, idx, val


def test_topk_spec_example(orc):
    # [0.1,-5,0.2,3], k=2 -> (1,-5), (3,3)
    p = orc.compress(C(orc, TOP_K, k_num=1, k_den=2), [0.1, -5, 0.2, 3])
    k, idx, val = _sparse(p)
    assert (k, idx, val) == (2, [1, 3], [-5.0, 3.0])
    assert list(orc.decompress(C(orc, TOP_K, k_num=1, k_den=2), p, 4)) == [0, -5, 0, 3]


def test_topk_k_resolution(orc):
    # R8: k = max(1, floor(L * num / den)) in integers ("k = 0.1%")
    c = C(orc, TOP_K, k_num=1, k_den=1000)
    assert orc.topk_k(c, 262144) == 262
    assert orc.topk_k(c, 999) == 1
    assert orc.topk_k(c, 2000) == 2
    assert orc.topk_k(C(orc, RANDOM_K, k_num=1, k_den=32), 1024) == 32


@pytest.mark.parametrize("d", [1, 2, 3, 4])
def test_topk_brute_force(orc, d):
    # exhaustive over {-2,-1,-0,0,1,2}^d: the chosen set S has |S| = k and every
    # i in S beats every j not in S in the order (|x| desc, index asc) (R9).
    vals = [-2.0, -1.0, -0.0, 0.0, 1.0, 2.0]
    for k in range(1, d + 1):
        c = C(orc, TOP_K, k_num=k, k_den=d)
        for x in itertools.product(vals, repeat=d):
            kk, idx, val = _sparse(orc.compress(c, list(x)))
            assert kk == k and idx == sorted(idx) and len(set(idx)) == k
            S = set(idx)
            for i in S:
                for j in range(d):
                    if j not in S:
                        assert abs(x[i]) > abs(x[j]) or (abs(x[i]) == abs(x[j]) and i < j)
            assert all(struct.pack("<f", v) == struct.pack("<f", x[i]) for i, v in zip(idx, val))


def test_topk_brute_force_random(orc):
    rng = np.random.default_rng(5)
    for trial in range(200):
        d = int(rng.integers(1, 40))
        x = np.round(rng.standard_normal(d) * 4) / 4  # many ties
        k = int(rng.integers(1, d + 1))
        _, idx, _ = _sparse(orc.compress(C(orc, TOP_K, k_num=k, k_den=d), x))
        order = sorted(range(d), key=lambda j: (-abs(float(np.float32(x[j]))), j))
        assert idx == sorted(order[:k])


def test_fused_ef_equivalence_topk(orc):
    # PAPER.md:501-502 / SPEC.md:176: e = q - dec(C(q)) equals q with the k
    # selected entries zero-filled, bit for bit.
    rng = np.random.default_rng(2)
    for d in (4, 100, 1001):
        q = rng.standard_normal(d).astype(np.float32)
        c = C(orc, TOP_K, k_num=1, k_den=10)
        p = orc.compress(c, q)
        e = q - orc.decompress(c, p, d)
        _, idx, _ = _sparse(p)
        z = q.copy()
        z[idx] = 0.0
        assert e.tobytes() == z.tobytes()
        assert np.array_equal(orc.decompress(c, p, d) + e, q)  # EF conservation, exact


def test_topk_rate_arithmetic(orc):
    # int32 indices + values. With fp32 values (R20) the rate vs
    # fp32 is 4e6 / (8 + 8000); the paper's 333x is 2e6 / (1000 * (4 + 2)).
    assert orc.payload_bytes(C(orc, TOP_K), 0, 10 ** 6) == 8 + 8 * 1000
    assert abs(2e6 / (1000 * (4 + 2)) - 333.33) < 0.01


# ---------------------------------------------------------------- random-k
def test_randomk_full_selection_is_identity(orc):
    # k = d keeps everything with scale d/k = 1
    x = np.float32([1.5, -2.25, 0, 3])
    for scaled in (0, 1):
        c = C(orc, RANDOM_K, k_num=1, k_den=1, randk_scaled=scaled)
        assert np.array_equal(orc.decompress(c, orc.compress(c, x, seed=9), 4), x)


def test_randomk_two_outcomes(orc):
    # d=2, k=1, x=[2,0] scaled: outcomes [4,0] or [0,0], each w.p. 1/2
    c = C(orc, RANDOM_K, k_num=1, k_den=2, randk_scaled=1)
    outs = [tuple(orc.decompress(c, orc.compress(c, [2, 0], seed=s, chunk=3, t=1), 2))
            for s in range(4000)]
    assert set(outs) == {(4.0, 0.0), (0.0, 0.0)}
    frac = sum(o == (4.0, 0.0) for o in outs) / len(outs)
    assert abs(frac - 0.5) < 4 * 0.5 / np.sqrt(len(outs))


def test_randomk_unbiased_and_uniform(orc):
    # Def. 1: E[C(x)] = x for the scaled estimator; each index kept w.p. k/d
    rng = np.random.default_rng(4)
    d, k, T = 16, 4, 6000
    x = rng.standard_normal(d).astype(np.float32)
    c = C(orc, RANDOM_K, k_num=k, k_den=d, randk_scaled=1)
    acc = np.zeros(d)
    cnt = np.zeros(d)
    for s in range(T):
        dec = orc.decompress(c, orc.compress(c, x, seed=12345, chunk=s, t=1), d).astype(np.float64)
        acc += dec
        cnt += dec != 0
    p = k / d
    se_cnt = np.sqrt(T * p * (1 - p))
    assert np.all(np.abs(cnt - T * p) < 4.5 * se_cnt)
    se = np.abs(x) * (d / k) * np.sqrt(p * (1 - p) / T)
    assert np.all(np.abs(acc / T - x) < 4.5 * se + 1e-7)


def test_randomk_drop_fraction(orc):
    # k = 1/32 drops exactly 96.875% of the entries
    c = C(orc, RANDOM_K, k_num=1, k_den=32)
    d = 32 * 1000
    x = np.ones(d, dtype=np.float32)
    dec = orc.decompress(c, orc.compress(c, x, seed=1), d)
    assert np.count_nonzero(dec == 0) / d == 0.96875


# ---------------------------------------------------------------- dithering
def test_linear_dither_zero_and_scalar(orc):
    for b in (2, 5, 7, 8):
        c = C(orc, LINEAR_DITHER, bits=b)
        assert np.array_equal(orc.decompress(c, orc.compress(c, np.zeros(9, np.float32)), 9), np.zeros(9))
        for v in (3.0, -0.125, 7.5e-5):
            assert orc.decompress(c, orc.compress(c, [v], seed=5), 1)[0] == np.float32(v)


def test_linear_dither_on_grid_deterministic(orc):
    # entries on the grid are reproduced exactly, for every seed
    c = C(orc, LINEAR_DITHER, bits=2)   # s = 1: grid {0, 1} of |x|/||x||
    for s in range(50):
        assert list(orc.decompress(c, orc.compress(c, [0, 0, -4, 0], seed=s), 4)) == [0, 0, -4, 0]


def test_linear_dither_spec_probabilities(orc):
    # bits=2 (s=1), x=[3,4]: 3/5 rounds up w.p. 0.6, 4/5 w.p. 0.8
    c = C(orc, LINEAR_DITHER, bits=2)
    T = 20000
    up = np.zeros(2)
    for s in range(T):
        dec = orc.decompress(c, orc.compress(c, [3, 4], seed=77, chunk=s, t=2), 2)
        assert set(np.abs(dec)).issubset({0.0, 5.0})
        up += dec == 5.0
    for frac, p in zip(up / T, (0.6, 0.8)):
        assert abs(frac - p) < 4 * np.sqrt(p * (1 - p) / T)


def test_natural_dither_spec_probability(orc):
    # bits=3, normalized 0.75 brackets 0.5 and 1.0, up w.p. 0.5.
    # x = [0.75, sqrt(1-0.75^2)] has ||x|| = 1 (up to fp32 rounding of N).
    c = C(orc, NATURAL_DITHER, bits=3)
    x = np.float32([0.75, np.sqrt(1 - 0.75 ** 2)])
    T = 20000
    up = 0
    for s in range(T):
        dec = orc.decompress(c, orc.compress(c, x, seed=3, chunk=s), 2)
        N = np.float32(np.sqrt(np.sum(x.astype(np.float64) ** 2)))
        assert dec[0] in (np.float32(0.5) * N, np.float32(1.0) * N)
        up += dec[0] == N
    assert abs(up / T - 0.5) < 4 * np.sqrt(0.25 / T)


def test_natural_dither_levels(orc):
    # R11: bits=3 levels {0, 1/4, 1/2, 1} of |x|/||x||; d=1 exact
    c = C(orc, NATURAL_DITHER, bits=3)
    for v in (2.0, -0.5):
        assert orc.decompress(c, orc.compress(c, [v]), 1)[0] == np.float32(v)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(64).astype(np.float32)
    N = np.float32(np.sqrt(np.sum(x.astype(np.float64) ** 2)))
    dec = orc.decompress(c, orc.compress(c, x, seed=11), 64)
    allowed = {0.0} | {float(np.float32(lv) * N) for lv in (0.25, 0.5, 1.0)}
    assert set(np.abs(dec).tolist()).issubset(allowed)


@pytest.mark.parametrize("kind,bits", [(LINEAR_DITHER, 2), (LINEAR_DITHER, 7), (NATURAL_DITHER, 3)])
def test_dither_unbiased(orc, kind, bits):
    # Def. 1: per-coordinate mean within 4.5 SE of x
    rng = np.random.default_rng(bits)
    d, T = 12, 20000
    x = (rng.standard_normal(d)).astype(np.float32)
    c = C(orc, kind, bits=bits)
    s1 = np.zeros(d)
    s2 = np.zeros(d)
    for s in range(T):
        dec = orc.decompress(c, orc.compress(c, x, seed=2024, chunk=s, t=1), d).astype(np.float64)
        s1 += dec
        s2 += dec * dec
    mean = s1 / T
    se = np.sqrt(np.maximum(s2 / T - mean ** 2, 0) / T)
    assert np.all(np.abs(mean - x) <= 4.5 * se + 2e-6 * np.abs(x) + 1e-7)


def test_dither_payload_sizes(orc):
    # [f32 norm][ceil(b*d/8) bytes]
    for b in range(2, 9):
        for kind in (LINEAR_DITHER, NATURAL_DITHER):
            assert orc.payload_bytes(C(orc, kind, bits=b), 0, 1001) == 4 + (b * 1001 + 7) // 8
    assert orc.payload_bytes(C(orc, NONE), 0, 10) == 40
    assert orc.payload_bytes(C(orc, SCALED_SIGN), 1, 10) == 40   # raw unit


def test_dither_code_packing(orc):
    # codes are `bits`-bit fields, LSB-first at bit offset bits*j;
    # code = sign | level << 1 with sign 1 = nonnegative
    c = C(orc, LINEAR_DITHER, bits=5)
    x = np.float32([0, 1, -1, 2, -2, 0.5, 3, -3, 1.5])
    p = orc.compress(c, x, seed=1)
    N = struct.unpack("<f", p[:4])[0]
    bitsint = int.from_bytes(p[4:], "little")
    dec = orc.decompress(c, p, 9)
    unit = np.float32(N) / np.float32(15)
    for j in range(9):
        code = (bitsint >> (5 * j)) & 31
        sign = code & 1
        assert sign == (0 if x[j] < 0 else 1)
        assert dec[j] == (1 if sign else -1) * np.float32(np.float32(code >> 1) * unit)


# ---------------------------------------------------------------- dithering: bit-exact vectors
def test_dither_golden_vectors(orc):
    # SURVEY.md:566-573 (tests/golden/dither_vectors.json): Philox words, codes and
    # packed bytes derived outside this repo; a change to the counter layout, the
    # word selection, u = (w >> 8) * 2^-24 or the code packing fails here even when
    # the output stays uniform / unbiased (which the statistical pins above allow).
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dither_vectors.json")))
    s = g["stream"]
    words = [orc.rng_word(s["seed"], j, s["chunk"], s["t"], s["stage"], s["rank"]) for j in range(8)]
    assert ["%08x" % w for w in words] == g["philox_words_w0_w7"]
    for case in g["cases"]:
        kind = LINEAR_DITHER if case["kind"] == "linear" else NATURAL_DITHER
        b = case["bits"]
        comp = C(orc, kind, bits=b, use_ef=0)
        x = np.array(case["x"], np.float32)
        p = orc.compress(comp, x, seed=s["seed"], chunk=s["chunk"], t=s["t"], stage=s["stage"], rank=s["rank"])
        assert p[:4].hex() == case["norm_f32_le"], case
        assert p[4:].hex() == case["packed"], case
        body = int.from_bytes(p[4:], "little")
        codes = [(body >> (b * j)) & ((1 << b) - 1) for j in range(len(x))]
        assert codes == case["codes"], case
        if "levels" in case and kind == LINEAR_DITHER:
            assert [c >> 1 for c in codes] == case["levels"]
        if kind == NATURAL_DITHER:
            cmax = (1 << (b - 1)) - 1
            lev = [0.0 if (c >> 1) == 0 else 2.0 ** -(cmax - (c >> 1)) for c in codes]
            assert lev == case["levels"]
        if "dec" in case:
            assert list(orc.decompress(comp, p, len(x))) == case["dec"]
