"""Per-tensor compression units on the GPU (NEXT #4: the paper
compresses whole tensors; `unit_mode = 1`, the oracle's chunk_elems = 0):
two-pass worker / server kernels with a per-unit pairwise tree over the slice
partials.  Units of 37 and 184 slices exercise trees beyond one warp; payloads
and errors bit-exact, m, v, x within 1e-6 relative."""
import pytest

from workloads import LINEAR_DITHER, NATURAL_DITHER, NONE, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config

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


SPARSE = [
    ("topk_ef", Comp(TOP_K, 1, 1000, use_ef=1)),
    ("topk_f16_ef", Comp(TOP_K, 1, 1000, use_ef=1, f16=1)),
    ("topk_noef", Comp(TOP_K, 1, 1000, use_ef=0)),
    ("randk_ef", Comp(RANDOM_K, 1, 32, use_ef=1)),
    ("randk_scaled", Comp(RANDOM_K, 1, 32, randk_scaled=1, use_ef=0)),
]


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("name,comp", SPARSE, ids=[k[0] for k in SPARSE])
def test_per_tensor_sparse(name, comp, n):
    # whole-tensor top-k / random-k: units of 300000 and
    # 1500000 elements take the large-unit path (multi-CTA radix select over the
    # candidates, ordered emission by slice count / scan / compaction)
    from gpu_harness import run_parity
    w = Config("units", "custom", comp, numels=SHAPES, chunk_elems=0)
    run_parity(w, n, steps=3, label=f"per-tensor {name} n={n}")


def test_per_tensor_sparse_p2p():
    from gpu_harness import run_parity
    w = Config("units", "custom", Comp(TOP_K, 1, 1000, use_ef=1, f16=1), numels=SHAPES, chunk_elems=0)
    run_parity(w, 2, steps=2, label="per-tensor topk p2p", mode="p2p")


@pytest.mark.slow
def test_per_tensor_topk_vgg_fc6():
    # VGG16 fc6 as one unit: 102,760,448 elements, k = 102,760 (top-k 0.1%, binary16
    # values as C3), against the oracle's whole-tensor selection
    from gpu_harness import run_parity
    w = Config("fc6", "custom", Comp(TOP_K, 1, 1000, use_ef=1, f16=1), numels=(102760448, 4096), chunk_elems=0)
    run_parity(w, 1, steps=2, label="per-tensor fc6")
