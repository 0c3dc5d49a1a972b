"""One whole step (A1-A9: compress, push, server, pull, update; PAPER.md:243-255,
Alg. 4-5) captured ONCE into a CUDA graph and replayed: the step counter t (the
bias corrections of R16, the Philox counter word of R13) and the launch /
exchange epochs live on the device (DevState, kernels.h) and advance inside the
kernels, so every replay is the next step.  Each replayed step is compared with
the oracle (payloads, e, e~ bit-exact; m, v, x within 1e-6) - at n = 1 and on a
bpc_connect_local peer group (the fused NVLink exchange's flags and waits inside
the graph)."""
import numpy as np
import pytest

from workloads import (LINEAR_DITHER, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config, gen_grad)

pytestmark = pytest.mark.gpu

SHAPES = (1000, 300000, 70000, 262147, 5)
KINDS = [
    ("onebit_ef", Comp(SCALED_SIGN, use_ef=1), "adam"),
    ("topk_ef", Comp(TOP_K, 1, 1000, use_ef=1), "adam"),
    ("randk_ef", Comp(RANDOM_K, 1, 32, use_ef=1), "adam"),
    ("ldither2_ef", Comp(LINEAR_DITHER, bits=2, use_ef=1), "adam"),
    ("onebit_lans", Comp(SCALED_SIGN, use_ef=1), "lans"),
    ("topk_nag", Comp(TOP_K, 1, 1000, use_ef=1), "nag"),
]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2105_07829_b200.build as b
    b.build()


def _issue(grp, grads, lr):
    """The step's calls in order, no host synchronisation (capturable)."""
    for i, c in enumerate(grp.ctxs):
        c.compress(grads[i])
    for c in grp.ctxs:
        c.exchange_push()
    for c in grp.ctxs:
        c.server()
    for c in grp.ctxs:
        c.exchange_pull()
    for i, c in enumerate(grp.ctxs):
        c.step(grp.x[i], lr)


def _run_graph(w, n, steps, lr, label, eager_after=0):
    import torch
    import oracle
    from gpu_harness import LoopbackGroup, compare_step, oracle_for
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):   # the contexts borrow s (context_for: current stream)
        grp = LoopbackGroup(w, n, mode="p2p" if n > 1 else "copy")
        ocfg, ost = oracle_for(w, n)
        gstat = [torch.zeros(grp.D, dtype=torch.float32, device="cuda") for _ in range(n)]
        try:
            def load(step):
                gs = [gen_grad(w, i, step) for i in range(n)]
                for i in range(n):
                    gstat[i].copy_(torch.from_numpy(gs[i]), non_blocking=False)
                return gs
            # step 1 eager (first-launch attributes), then capture
            gs = load(1)
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), lr)
            _issue(grp, gstat, lr)
            s.synchronize()
            compare_step(grp, ocfg, ost, delta, p, label=f"{label} eager step 1")
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                _issue(grp, gstat, lr)
            assert grp.ctxs[0].t == 2, "capture must not advance t"
            step = 1
            for _ in range(steps):
                step += 1
                gs = load(step)
                delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), lr)
                g.replay()
                s.synchronize()
                compare_step(grp, ocfg, ost, delta, p, label=f"{label} replay step {step}")
                assert all(c.t == step + 1 for c in grp.ctxs), "t after replay"
            for _ in range(eager_after):   # eager calls continue the replayed sequence
                step += 1
                gs = load(step)
                delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), lr)
                _issue(grp, gstat, lr)
                s.synchronize()
                compare_step(grp, ocfg, ost, delta, p, label=f"{label} eager step {step}")
            for c in grp.ctxs:
                c.sync()
        finally:
            s.synchronize()
            grp.close()


@pytest.mark.parametrize("name,comp,opt", KINDS, ids=[k[0] for k in KINDS])
def test_graph_replay_n1(name, comp, opt):
    w = Config("graph", "custom", comp, numels=SHAPES, optimizer=opt, lr=1e-2 if opt == "lans" else 1e-3)
    _run_graph(w, 1, steps=3, lr=w.lr, label=f"graph {name}", eager_after=1)


@pytest.mark.parametrize("name,comp,opt", KINDS[:4], ids=[k[0] for k in KINDS[:4]])
def test_graph_replay_p2p_group(name, comp, opt):
    w = Config("graph", "custom", comp, numels=SHAPES, optimizer=opt)
    _run_graph(w, 2, steps=3, lr=w.lr, label=f"graph p2p {name}", eager_after=1)


def test_graph_replay_per_tensor_units():
    w = Config("graph", "custom", Comp(SCALED_SIGN, use_ef=1), numels=(1000, 70000, 300000, 1500000, 5),
               chunk_elems=0)
    _run_graph(w, 2, steps=2, lr=w.lr, label="graph per-tensor", eager_after=0)


def test_set_step_moves_device_counter():
    import torch
    import paper_2105_07829_b200 as bpc
    w = Config("graph", "custom", Comp(SCALED_SIGN, use_ef=1), numels=SHAPES)
    c = bpc.context_for(w, rank=0, world_size=1)
    try:
        assert c.t == 1
        c.set_step(12345)
        assert c.t == 12345
        with pytest.raises(bpc.BpcError):
            c.set_step(0)
        assert c.t == 12345
    finally:
        torch.cuda.synchronize()
        c.finalize()
