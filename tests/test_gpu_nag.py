"""NAG update (reading R24; the optimizer of the paper's CNN runs)
on the CUDA path vs the oracle: velocity (in m) and x bit-exact by
construction (bar 1e-6 relative), payloads and errors bit-exact."""
import pytest

from workloads import LINEAR_DITHER, NONE, SCALED_SIGN, TOP_K, Comp, Config

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("topk_f16_ef", Comp(TOP_K, 1, 1000, use_ef=1, f16=1)),
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
def test_nag_parity(name, comp, n):
    from gpu_harness import run_parity
    w = Config("nag", "custom", comp, numels=SHAPES, optimizer="nag", momentum=0.9, lr=0.1)
    run_parity(w, n, steps=3, label=f"nag {name} n={n}")


def test_nag_rejects_bad_momentum():
    import paper_2105_07829_b200 as bpc
    w = Config("nag", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES, optimizer="nag", momentum=1.0)
    with pytest.raises(bpc.BpcError):
        bpc.context_for(w)
