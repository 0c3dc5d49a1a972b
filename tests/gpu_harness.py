"""Test-only drivers that run the CUDA path (through the C ABI) beside the oracle.

`LoopbackGroup` drives n ranks' libbpc contexts on ONE GPU.
* mode "copy": the all-to-all / all-gather are device copies through the
  buffer API (the external-exchange mode of bpc.h) - the analogue of SPEC's
  in-process transport;
* mode "p2p": the contexts are wired with bpc_connect_local into one peer-memory
  exchange group, so the product transport runs - the fused stores into the
  owners' RECV, the release / acquire flags, the update's bulk reads of the
  owners' P (norm-based kinds), the copy + wait kernels (sparse kinds) - with
  every phase issued for all ranks before the next on one shared stream.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2105_07829_b200 as bpc
from workloads import Config, gen_grad, gen_params, layout


class LoopbackGroup:
    def __init__(self, wcfg: Config, n: int, device: int = 0, mode: str = "copy"):
        self.w = wcfg
        self.n = n
        self.numels = wcfg.tensor_numels()
        self.offs, self.D = layout(self.numels)
        self.ctxs = [bpc.context_for(wcfg, rank=r, world_size=n, device=device, check_finite=1)
                     for r in range(n)]
        self.mode = mode if n > 1 else "copy"
        if self.mode == "p2p":
            bpc.connect_local(self.ctxs)
            assert all(c.exchange == "p2p" for c in self.ctxs)
        # fused exchange (norm-based kinds over p2p): SEND is never written and P
        # holds only the owner's segment
        self.fused = self.mode == "p2p" and wcfg.comp.kind not in (3, 4)
        self.x = [torch.tensor(gen_params(wcfg), device="cuda") for _ in range(n)]

    def step(self, grads, lr, sync=True):
        n, ctxs = self.n, self.ctxs
        for i, c in enumerate(ctxs):
            c.compress(grads[i])
        if self.mode == "p2p":
            for c in ctxs:
                c.exchange_push()
            for c in ctxs:
                c.server()
            for c in ctxs:
                c.exchange_pull()
            for i, c in enumerate(ctxs):
                c.step(self.x[i], lr)
            if sync:
                for c in ctxs:
                    c.sync()
            return
        if n > 1:
            for r in range(n):
                recv = ctxs[r].buffer(bpc.BUF_RECV)
                slot = ctxs[r].summary().recv_slot_bytes
                for i in range(n):
                    off, b = ctxs[i].peer_segment(r)
                    assert b == slot
                    if b:
                        recv[i * slot:(i + 1) * slot].copy_(ctxs[i].buffer(bpc.BUF_SEND)[off:off + b])
        for c in ctxs:
            c.exchange_push()
        for c in ctxs:
            c.server()
        if n > 1:
            for r in range(n):
                off, b = ctxs[r].peer_segment(r)
                src = ctxs[r].buffer(bpc.BUF_P)[off:off + b]
                for i in range(n):
                    if i != r and b:
                        ctxs[i].buffer(bpc.BUF_P)[off:off + b].copy_(src)
        for c in ctxs:
            c.exchange_pull()
        for i, c in enumerate(ctxs):
            c.step(self.x[i], lr)
        for c in ctxs:
            c.sync()

    def close(self):
        for c in self.ctxs:
            c.finalize()


def oracle_for(wcfg: Config, n: int):
    cfg = oracle.Cfg.from_workload(wcfg, n=n)
    offs, D = layout(wcfg.tensor_numels())
    st = oracle.State(n, D, gen_params(wcfg))
    return cfg, st


def f32(a: np.ndarray) -> np.ndarray:
    return np.frombuffer(a.tobytes(), dtype=np.float32)


class Mismatch(AssertionError):
    pass


def compare_step(grp: LoopbackGroup, ocfg, ost, delta, p, *, label=""):
    """Compare every chunk's payloads (bit-exact), e, e~ (bit-exact) and m, v, x.
    Worker payloads are read where the exchange left them: SEND, and the owner's
    RECV slot (n > 1); server payloads in every rank's P, or only in the owner's
    P for the fused exchange (the update reads it there over peer memory)."""
    n = grp.n
    lay = ocfg.payload_layout()
    plan = ocfg.plan()
    fused = getattr(grp, "fused", False)
    sends = [c.copy_state(bpc.BUF_SEND) for c in grp.ctxs]
    pbufs = [c.copy_state(bpc.BUF_P) for c in grp.ctxs]
    recvs = [c.copy_state(bpc.BUF_RECV) for c in grp.ctxs] if n > 1 else None
    slots = [c.summary().recv_slot_bytes for c in grp.ctxs]
    chunks = grp.ctxs[0].chunks()
    assert len(chunks) == len(plan), "chunk plans differ"
    for ci, (ti, off, L, raw) in enumerate(plan):
        gc = chunks[ci]
        assert (gc.tensor, gc.offset, gc.len, gc.raw) == (ti, off, L, raw), f"chunk {ci} plan"
        po, pb = lay[ci]
        assert gc.payload_bytes == pb, f"chunk {ci} payload size"
        for i in range(n):
            o = delta[i, po:po + pb]
            got = []
            if not fused:
                got.append(("SEND", sends[i][gc.payload_offset:gc.payload_offset + pb]))
            if n > 1:   # as received by the owner, slot i
                ro = i * slots[gc.owner] + gc.recv_offset
                got.append(("RECV", recvs[gc.owner][ro:ro + pb]))
            for where, g in got:
                if g.tobytes() != o.tobytes():
                    bad = np.nonzero(g != o)[0]
                    raise Mismatch(f"{label} worker {i} chunk {ci} (L={L}, raw={raw}) payload in {where} differs "
                                   f"at {bad[:8]} of {pb} bytes")
        for i in range(n):   # after the all-gather every rank holds every p (fused: the owner's P)
            if fused and i != gc.owner:
                continue
            g = pbufs[i][gc.payload_offset:gc.payload_offset + pb]
            if g.tobytes() != p[po:po + pb].tobytes():
                bad = np.nonzero(g != p[po:po + pb])[0]
                raise Mismatch(f"{label} rank {i} server payload of chunk {ci} (L={L}) differs at "
                               f"{bad[:8]} of {pb} bytes")
    # worker errors
    for i in range(n):
        e = f32(grp.ctxs[i].copy_state(bpc.BUF_WORKER_ERR))
        for ci, (ti, off, L, raw) in enumerate(plan):
            if e[off:off + L].tobytes() != ost.e[i, off:off + L].tobytes():
                d = np.nonzero(e[off:off + L] != ost.e[i, off:off + L])[0]
                raise Mismatch(f"{label} worker error e_{i} chunk {ci} differs at {d[:8]}")
    # server errors (owner only)
    etl = [f32(c.copy_state(bpc.BUF_SERVER_ERR)) for c in grp.ctxs]
    for ci, (ti, off, L, raw) in enumerate(plan):
        gc = chunks[ci]
        if raw or not grp.w.comp.use_ef:
            continue
        owner_info = grp.ctxs[gc.owner].chunk(ci)
        s0 = owner_info.server_err_offset
        got = etl[gc.owner][s0:s0 + L]
        if got.tobytes() != ost.et[off:off + L].tobytes():
            d = np.nonzero(got != ost.et[off:off + L])[0]
            raise Mismatch(f"{label} server error chunk {ci} differs at {d[:8]}")
    # optimizer state, parameters: identical on every rank (worker symmetry)
    m = f32(grp.ctxs[0].copy_state(bpc.BUF_M))
    v = f32(grp.ctxs[0].copy_state(bpc.BUF_V))
    xs = [grp.x[i].cpu().numpy() for i in range(n)]
    for i in range(1, n):
        assert xs[i].tobytes() == xs[0].tobytes(), "parameters differ between ranks"
    for name, got, want in (("m", m, ost.m), ("v", v, ost.v), ("x", xs[0], ost.x)):
        for ci, (ti, off, L, raw) in enumerate(plan):
            a, b = got[off:off + L], want[off:off + L]
            if a.tobytes() != b.tobytes():
                rel = np.max(np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b), 1e-30))
                if rel > 1e-6:
                    raise Mismatch(f"{label} {name} chunk {ci} rel diff {rel:.3e} > 1e-6")


def run_parity(wcfg: Config, n: int, steps: int, lr: float = 1e-3, label="", mode="copy"):
    grp = LoopbackGroup(wcfg, n, mode=mode)
    ocfg, ost = oracle_for(wcfg, n)
    try:
        for step in range(1, steps + 1):
            gs = [gen_grad(wcfg, i, step) for i in range(n)]
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), lr)
            grp.step([torch.tensor(g, device="cuda") for g in gs], lr)
            compare_step(grp, ocfg, ost, delta, p, label=f"{label} step {step}")
    finally:
        grp.close()
