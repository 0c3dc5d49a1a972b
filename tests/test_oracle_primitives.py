"""Pins for the oracle's primitives: Philox4x32-10 and the fp64 pairwise sum.

Each check compares the oracle against something other than itself: the
Random123 published known-answer vectors, hand-worked sums whose value the
definition (R6) fixes, and the exact sum (math.fsum) within the
textbook pairwise-summation error bound.
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.filterwarnings("ignore")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kats():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(x, 16) for x in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kats())
def test_philox_random123_kat(orc, ctr, key, out):
    assert orc.philox(ctr, key) == out


def test_rng_word_counter_layout(orc):
    # R13: word j%4 of Philox((j//4, chunk, t, stage<<31|rank), (lo32 seed, hi32 seed))
    seed = 0x0123456789ABCDEF
    for j in (0, 1, 5, 4099):
        for (chunk, t, stage, rank) in ((0, 1, 0, 0), (7, 3, 1, 0), (2, 9, 0, 5)):
            words = orc.philox([j // 4, chunk, t, (stage << 31) | rank],
                               [seed & 0xFFFFFFFF, seed >> 32])
            assert orc.rng_word(seed, j, chunk, t, stage, rank) == words[j % 4]


def test_pairwise_hand_examples(orc):
    # [1, 0, 2^-53, 2^-53]: pairwise (1+0) + (2^-53+2^-53) = 1 + 2^-52, while a
    # left-to-right sum gives 1 (each 2^-53 is a tie that rounds to even).
    t = 2.0 ** -53
    assert orc.pairwise_sum([1.0, 0.0, t, t]) == 1.0 + 2.0 ** -52
    # [t, t, 1, 0] also 1 + 2^-52; [1, t, t, 0] gives (1+t)+(t+0) = 1 + t -> 1
    assert orc.pairwise_sum([t, t, 1.0, 0.0]) == 1.0 + 2.0 ** -52
    assert orc.pairwise_sum([1.0, t, t, 0.0]) == 1.0
    # odd length pads with +0: [1, t, t] -> (1 + t) + (t + 0) = 1
    assert orc.pairwise_sum([1.0, t, t]) == 1.0
    assert orc.pairwise_sum([]) == 0.0
    assert orc.pairwise_sum([3.5]) == 3.5


def test_pairwise_exact_on_integers(orc):
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 7, 8, 100, 4097):
        a = rng.integers(0, 1000, size=n).astype(np.float64)
        assert orc.pairwise_sum(a) == float(a.sum())


@pytest.mark.parametrize("n", [5, 128, 1000, 1 << 14, (1 << 16) + 3])
def test_pairwise_within_error_bound(orc, n):
    rng = np.random.default_rng(n)
    a = np.abs(rng.standard_normal(n)) * 10.0 ** rng.uniform(-6, 3, size=n)
    exact = math.fsum(a)
    got = orc.pairwise_sum(a)
    # pairwise summation: |err| <= ceil(log2 n) * u * sum|a| (Higham, ASNA §4.2)
    bound = math.ceil(math.log2(n)) * 2.0 ** -53 * float(np.sum(np.abs(a))) * 1.01
    assert abs(got - exact) <= bound


def test_pairwise_padding_invariance(orc):
    # padding with zeros to any larger power of two leaves the value unchanged
    rng = np.random.default_rng(3)
    a = np.abs(rng.standard_normal(300))
    s = orc.pairwise_sum(a)
    for extra in (212, 724, 1748):
        assert orc.pairwise_sum(np.concatenate([a, np.zeros(extra)])) == s
