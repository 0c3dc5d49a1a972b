"""Pins of the oracle's binary16 sparse values (NEXT #4, reading R23): the
top-k / random-k payload [u64 k][k x u32 index][k x f16 value] of the paper's
333x rate, checked against numpy's float32 -> float16
conversion (a library routine) and the closed-form payload size."""
import numpy as np
import pytest

import oracle
from workloads import RANDOM_K, TOP_K, Comp


def parse(payload, L, f16):
    b = np.frombuffer(payload, dtype=np.uint8)
    k = int(b[:8].view(np.uint64)[0])
    idx = b[8:8 + 4 * k].view(np.uint32)
    vb = b[8 + 4 * k:]
    val = vb[:2 * k].view(np.float16).astype(np.float32) if f16 else vb[:4 * k].view(np.float32)
    return k, idx, val


@pytest.mark.parametrize("L", [1 << 18, 1 << 20])
def test_rate_333(L):
    # top-k 0.1% with 16-bit values and 32-bit indices is 333x
    # smaller than the fp16 gradient
    comp = Comp(TOP_K, 1, 1000, f16=1)
    k = oracle.topk_k(comp, L)
    assert oracle.payload_bytes(comp, 0, L) == 8 + 6 * k
    assert 2 * L / (6 * k) == pytest.approx(333.3, rel=3e-3)


@pytest.mark.parametrize("kind", [TOP_K, RANDOM_K])
def test_values_are_numpy_float16(kind):
    rng = np.random.default_rng(7)
    L = 5000
    x = (rng.standard_normal(L) * 10 ** rng.uniform(-6, 3, L)).astype(np.float32)
    for f16 in (0, 1):
        comp = Comp(kind, 1, 20, f16=f16, randk_scaled=1 if kind == RANDOM_K else 0)
        k, idx, val = parse(oracle.compress(comp, x, seed=3, chunk=2, t=5), L, f16)
        if f16 == 0:
            idx32, val32 = idx.copy(), val.copy()
    assert np.array_equal(idx, idx32)                       # selection is on the fp32 values
    want = np.clip(val32, -65504, 65504).astype(np.float16).astype(np.float32)
    assert val.tobytes() == want.tobytes()
    dec = oracle.decompress(comp, bytes(oracle.compress(comp, x, seed=3, chunk=2, t=5)), L)
    full = np.zeros(L, dtype=np.float32)
    full[idx] = want
    assert dec.tobytes() == full.tobytes()


def test_saturation_and_rounding():
    x = np.array([7.0e4, -1.0e5, 0.1, 1e-8, 65519.0, -0.0, 3.0], dtype=np.float32)
    comp = Comp(TOP_K, 1, 1, f16=1)                          # k = L: every value kept
    k, idx, val = parse(oracle.compress(comp, x), x.size, 1)
    assert k == x.size and list(idx) == list(range(x.size))
    np.testing.assert_array_equal(val, np.array([65504, -65504, 0.0999755859375, 0.0, 65504, -0.0, 3.0],
                                                dtype=np.float32))
