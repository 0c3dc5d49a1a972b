"""Real multi-GPU parity: one process per GPU (torchrun), libbpc's exchange
(bpc_aggregate; argv[2] = "p2p" NVLink peer stores or "nccl"), every rank
checked against the CPU oracle on the same seeded inputs.  argv[3] = "graph":
steps 5-8 replay a CUDA graph of one whole step captured after step 4 (the
step counter and exchange epochs advance on the device).  Launched by
tests/test_gpu_multi.py; prints "RANK <r> <case> OK" per rank and case."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import oracle
import paper_2105_07829_b200 as bpc
from workloads import (LINEAR_DITHER, RANDOM_K, SCALED_SIGN, TOP_K, Comp, Config, gen_grad, gen_params,
                       layout)

CASES = {
    "onebit": Comp(SCALED_SIGN, use_ef=1),
    "topk": Comp(TOP_K, 1, 1000, use_ef=1),
    "randk": Comp(RANDOM_K, 1, 32, use_ef=1),
    "ldither": Comp(LINEAR_DITHER, bits=7, use_ef=0),
    "lans_onebit": Comp(SCALED_SIGN, use_ef=1),   # + the LANS update (NEXT #1)
    "lans_topk": Comp(TOP_K, 1, 1000, use_ef=1),
    "units_onebit": Comp(SCALED_SIGN, use_ef=1),   # per-tensor units (two-pass kernels)
    "nag_topk": Comp(TOP_K, 1, 1000, use_ef=1, f16=1),
}
SHAPES = (1000, 300000, 70000, 262147, 5, 600000)


def f32(a):
    return np.frombuffer(a.tobytes(), dtype=np.float32)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] else list(CASES)
    exchange = sys.argv[2] if len(sys.argv) > 2 else "p2p"
    use_graph = len(sys.argv) > 3 and sys.argv[3] == "graph"
    stream = torch.cuda.Stream(dev)   # capturable: the contexts borrow it
    torch.cuda.set_stream(stream)
    for name in names:
        w = Config("mg", "custom", CASES[name], numels=SHAPES, n=world,
                   optimizer="lans" if name.startswith("lans") else "nag" if name.startswith("nag") else "adam",
                   chunk_elems=0 if name.startswith("units") else 1 << 18)
        offs, D = layout(w.tensor_numels())
        obj = [bpc.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = bpc.context_for(w, rank=rank, world_size=world, device=local, nccl_id=obj[0], check_finite=1,
                              exchange=exchange)
        sparse = name in ("topk", "randk", "lans_topk", "nag_topk")
        # NVLS applies to the fused kinds; the sparse kinds keep the peer copies
        want = "p2p" if (exchange == "nvls" and sparse) else exchange
        assert ctx.exchange == want, f"rank {rank}: asked for {exchange}, got {ctx.exchange}"
        x = torch.tensor(gen_params(w), device=dev)
        ocfg = oracle.Cfg.from_workload(w, n=world)
        ost = oracle.State(world, D, gen_params(w))
        lay = ocfg.payload_layout()
        plan = ocfg.plan()
        # steps 1-3 are checked one by one; steps 4-8 run back to back without a
        # host sync (ranks drift apart: the exchange's cross-step ordering), then
        # step 8 is checked
        dgrads = {step: torch.tensor(gen_grad(w, rank, step), device=dev) for step in range(4, 9)}
        gstat = torch.zeros(D, dtype=torch.float32, device=dev)
        graph = None
        torch.cuda.synchronize()
        for step in range(1, 9):
            gs = [gen_grad(w, i, step) for i in range(world)]
            delta, p, _ = oracle.round_(ocfg, ost, np.stack(gs), w.lr)
            if graph is not None:
                gstat.copy_(dgrads[step])
                graph.replay()
            else:
                ctx.compress(dgrads[step] if step in dgrads else torch.tensor(gs[rank], device=dev))
                ctx.aggregate()
                ctx.step(x, w.lr)
            if use_graph and step == 4:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    ctx.compress(gstat)
                    ctx.aggregate()
                    ctx.step(x, w.lr)
            if step not in (1, 2, 3, 8):
                continue
            ctx.sync()
            send = ctx.copy_state(bpc.BUF_SEND)
            recv = ctx.copy_state(bpc.BUF_RECV)
            slot = ctx.summary().recv_slot_bytes
            # the fused exchange (p2p, norm-based kinds) stores payloads straight into the
            # owners' RECV and never writes SEND
            check_send = exchange == "nccl" or sparse
            # ... and leaves p in its owner's P (the update kernels read it over NVLink),
            # except NVLS, which multicasts it into every rank's P
            check_all_p = check_send or exchange == "nvls"
            pb = ctx.copy_state(bpc.BUF_P)
            e = f32(ctx.copy_state(bpc.BUF_WORKER_ERR))
            etl = f32(ctx.copy_state(bpc.BUF_SERVER_ERR))
            xs = x.cpu().numpy()
            for ci, (ti, off, L, raw) in enumerate(plan):
                gc = ctx.chunk(ci)
                po, nb = lay[ci]
                if check_send:
                    assert send[gc.payload_offset:gc.payload_offset + nb].tobytes() == delta[rank, po:po + nb].tobytes(), \
                        f"{name} rank {rank} step {step}: worker payload of chunk {ci} differs"
                if gc.owner == rank:   # every rank's delta, as received by this owner
                    for r in range(world):
                        got = recv[r * slot + gc.recv_offset:r * slot + gc.recv_offset + nb]
                        assert got.tobytes() == delta[r, po:po + nb].tobytes(), \
                            f"{name} rank {rank} step {step}: received payload of rank {r}, chunk {ci} differs"
                if check_all_p or gc.owner == rank:
                    assert pb[gc.payload_offset:gc.payload_offset + nb].tobytes() == p[po:po + nb].tobytes(), \
                        f"{name} rank {rank} step {step}: server payload of chunk {ci} differs (owner {gc.owner})"
                assert e[off:off + L].tobytes() == ost.e[rank, off:off + L].tobytes(), \
                    f"{name} rank {rank} step {step}: worker error of chunk {ci} differs"
                if gc.owner == rank and not raw and w.comp.use_ef:
                    s0 = gc.server_err_offset
                    assert etl[s0:s0 + L].tobytes() == ost.et[off:off + L].tobytes(), \
                        f"{name} rank {rank} step {step}: server error of chunk {ci} differs"
                a, bref = xs[off:off + L], ost.x[off:off + L]
                rel = np.max(np.abs(a.astype(np.float64) - bref) / np.maximum(np.abs(bref), 1e-30))
                assert rel <= 1e-6, f"{name} rank {rank}: x rel diff {rel}"
        if use_graph:
            assert ctx.t == 9, f"rank {rank}: t = {ctx.t} after 8 steps"
        ctx.sync()
        graph = None
        ctx.finalize()
        dist.barrier()
        print(f"RANK {rank} {name} OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
