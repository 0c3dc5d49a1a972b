"""LANS / CLAN update (NEXT #1, reading R22) on the CUDA path vs the oracle.

Two streaming passes (m, v + per-tile pairwise block sums; x) and one CTA per
block for the coefficients; x, m, v compared at the north star's 1e-6 relative
(bit-exact by construction), payloads and errors bit-exact as in every parity
test.  Blocks = tensors: raw tensors (1000, 70000), multi-chunk / multi-tile
tensors with ragged tails (300000, 262147), a 5-element tensor; ||x_b|| is
below, inside and above the phi clamp."""
import pytest

from workloads import LINEAR_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("topk_ef", Comp(TOP_K, 1, 1000, use_ef=1)),
    ("randk_ef", Comp(RANDOM_K, 1, 32, use_ef=1)),
    ("ldither7", Comp(LINEAR_DITHER, bits=7, use_ef=0)),
    ("none", Comp(NONE, use_ef=1)),
]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("name,comp", KINDS, ids=[k[0] for k in KINDS])
def test_lans_parity(name, comp, n):
    from gpu_harness import run_parity
    w = Config("lans", "custom", comp, numels=SHAPES, optimizer="lans", lr=1e-2)
    run_parity(w, n, steps=3, label=f"lans {name} n={n}")


def test_lans_clamp_bounds():
    # alpha_l above every block norm: phi = alpha_l everywhere
    from gpu_harness import run_parity
    w = Config("lans", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES, optimizer="lans",
               alpha_l=20.0, alpha_u=30.0, lr=1e-3)
    run_parity(w, 1, steps=2, label="lans clamp")


def test_lans_rejects_bad_config():
    import paper_2105_07829_b200 as bpc
    w = Config("lans", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES, optimizer="lans",
               alpha_l=2.0, alpha_u=1.0)
    with pytest.raises(bpc.BpcError):
        bpc.context_for(w)
