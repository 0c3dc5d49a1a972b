"""Per-tensor compression units on the GPU (NEXT #4: the paper
compresses whole tensors; `unit_mode = 1`, the oracle's chunk_elems = 0):
two-pass worker / server kernels with a per-unit pairwise tree over the slice
partials.  Units of 37 and 184 slices exercise trees beyond one warp; payloads
and errors bit-exact, m, v, x within 1e-6 relative."""
import pytest

from workloads import LINEAR_DITHER, NATURAL_DITHER, NONE, SCALED_SIGN, TOP_K, Comp, Config

pytestmark = pytest.mark.gpu

SHAPES = (1000, 70000, 300000, 1500000, 5)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1)),
    ("ldither7", Comp(LINEAR_DITHER, bits=7, use_ef=0)),
    ("ndither3_ef", Comp(NATURAL_DITHER, bits=3, use_ef=1)),
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
def test_per_tensor_units(name, comp, n):
    from gpu_harness import run_parity
    w = Config("units", "custom", comp, numels=SHAPES, chunk_elems=0)
    run_parity(w, n, steps=3, label=f"per-tensor {name} n={n}")


def test_per_tensor_lans():
    from gpu_harness import run_parity
    w = Config("units", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES, chunk_elems=0, optimizer="lans",
               lr=1e-2)
    run_parity(w, 2, steps=2, label="per-tensor lans")


def test_per_tensor_rejects_topk():
    import paper_2105_07829_b200 as bpc
    w = Config("units", "custom", Comp(TOP_K, 1, 1000, use_ef=1), numels=SHAPES, chunk_elems=0)
    with pytest.raises(bpc.BpcError):
        bpc.context_for(w)
