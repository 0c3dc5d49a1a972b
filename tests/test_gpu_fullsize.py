"""Full-size parity at BASELINE.json's shapes (ResNet-50, VGG16, BERT-base,
BERT-large gradients, n = 1, the launch configuration bench.py times):
every unit's payload bytes, the worker and server errors, and m, v, x compared
with the CPU oracle element by element for two steps.  These runs push
thousands of slices through each persistent CTA, mixing raw and multi-slice
units, which is what exercises the pipelines' cross-CTA waits."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_fullsize_n1(name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import oracle
    from gpu_harness import LoopbackGroup, compare_step, oracle_for
    from workloads import config, gen_grad
    w = config(name, n=1)
    grp = LoopbackGroup(w, 1)
    ocfg, ost = oracle_for(w, 1)
    try:
        for step in (1, 2):
            g = gen_grad(w, 0, step)
            delta, p, _ = oracle.round_(ocfg, ost, g[None], w.lr)
            grp.step([torch.tensor(g, device="cuda")], w.lr)
            compare_step(grp, ocfg, ost, delta, p, label=f"{name} step {step}")
    finally:
        grp.close()


@pytest.mark.parametrize("name,n", [("C2", 2), ("C4", 2), ("C3", 2)])
def test_scaled_multi_rank(name, n):
    """Weak-scaled shapes (1/4 of every tensor) with n ranks on one GPU."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from gpu_harness import run_parity
    from workloads import config
    w = config(name, n=n, scale=4)
    run_parity(w, n, steps=2, label=f"{name}/4 n={n}")
