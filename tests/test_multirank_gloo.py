"""The N>1 exchange path on CPU: two and four processes over torch.distributed (gloo)
run the sharded server with libbpc's host plan (owner map, per-peer segments,
receive-slot offsets) and the oracle's per-unit operators, exchanging the
payload bytes with a real all-to-all and all-gather.  The decoded g~ must equal
the oracle's single-process round bit for bit: this pins the layout that
bpc_exchange_push / bpc_exchange_pull move over NCCL on the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import LINEAR_DITHER, SCALED_SIGN, TOP_K, Comp, Config, gen_grad, gen_params, layout

SHAPES = (1000, 300000, 70000, 262147, 5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, comp_t, steps, q):
    try:
        import oracle
        import paper_2105_07829_b200 as bpc
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comp = Comp(*comp_t)
        w = Config("gloo", "custom", comp, numels=SHAPES, n=world)
        numels = w.tensor_numels()
        offs, D = layout(numels)
        cfg = bpc.make_config(numels, offs, comp, world_size=world, rank=rank, seed=w.seed,
                              chunk_elems=w.chunk_elems, threshold_bytes=w.threshold_bytes)
        summ, chunks = bpc.plan(cfg)
        ocfg = oracle.Cfg.from_workload(w, n=world)
        ost = oracle.State(world, D, gen_params(w))
        oc = ocfg.s.comp
        e = np.zeros(D, np.float32)          # this worker's error
        et = np.zeros(D, np.float32)         # server error (owned chunks only)
        segs = []
        for r in range(world):
            mine = [c for c in chunks if c.owner == r]
            off = mine[0].payload_offset if mine else 0
            segs.append((off, sum((c.payload_bytes + 4 + 15) // 16 * 16 for c in mine)))
        assert summ.recv_slot_bytes == segs[rank][1]
        for step in range(1, steps + 1):
            g = gen_grad(w, rank, step)
            # ---- worker: payloads at the plan's offsets (SEND)
            send = np.zeros(summ.send_bytes, np.uint8)
            for ci, c in enumerate(chunks):
                sl = slice(c.offset, c.offset + c.len)
                ef = comp.use_ef and not c.raw
                qv = (g[sl] + e[sl]) if ef else g[sl].copy()
                pl = oracle.compress(oc, qv, raw=c.raw, seed=w.seed, chunk=ci, t=step, stage=0, rank=rank)
                send[c.payload_offset:c.payload_offset + len(pl)] = np.frombuffer(pl, np.uint8)
                if ef:
                    e[sl] = qv - oracle.decompress(oc, pl, c.len)
            # ---- all-to-all: segment r of SEND -> RECV slot `rank` of owner r
            slot = segs[rank][1]
            recv = torch.zeros(world * slot, dtype=torch.uint8)
            dist.all_to_all_single(recv, torch.from_numpy(send[:sum(b for _, b in segs)]),
                                   output_split_sizes=[slot] * world,
                                   input_split_sizes=[b for _, b in segs])
            recv = recv.numpy()
            # ---- server for owned chunks (Alg. 4 l.10-13): P segment
            pbuf = np.zeros(summ.send_bytes, np.uint8)
            for ci, c in enumerate(chunks):
                if c.owner != rank:
                    continue
                acc = np.zeros(c.len)
                for i in range(world):
                    base = i * slot + c.recv_offset
                    acc += oracle.decompress(oc, recv[base:base + c.payload_bytes].tobytes(), c.len, raw=c.raw)
                ef = comp.use_ef and not c.raw
                sl = slice(c.offset, c.offset + c.len)
                delta = (acc * (1.0 / world) + (et[sl].astype(np.float64) if ef else 0.0)).astype(np.float32)
                pl = oracle.compress(oc, delta, raw=c.raw, seed=w.seed, chunk=ci, t=step, stage=1, rank=0)
                pbuf[c.payload_offset:c.payload_offset + len(pl)] = np.frombuffer(pl, np.uint8)
                if ef:
                    et[sl] = delta - oracle.decompress(oc, pl, c.len)
            # ---- all-gather of the owners' P segments
            mx = max(b for _, b in segs)
            mine = torch.zeros(mx, dtype=torch.uint8)
            o, b = segs[rank]
            mine[:b] = torch.from_numpy(pbuf[o:o + b])
            got = [torch.zeros(mx, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(got, mine)
            for r, (o, b) in enumerate(segs):
                pbuf[o:o + b] = got[r].numpy()[:b]
            gt = np.zeros(D, np.float32)
            for ci, c in enumerate(chunks):
                gt[c.offset:c.offset + c.len] = oracle.decompress(oc, pbuf[c.payload_offset:c.payload_offset + c.payload_bytes].tobytes(), c.len, raw=c.raw)
            # ---- single-process oracle round on the same inputs
            _, _, ogt = oracle.round_(ocfg, ost, np.stack([gen_grad(w, i, step) for i in range(world)]), 0.0,
                                      want_payloads=False)
            for c in chunks:
                sl = slice(c.offset, c.offset + c.len)
                assert gt[sl].tobytes() == ogt[sl].tobytes(), f"rank {rank} step {step}: g~ differs"
                assert e[sl].tobytes() == ost.e[rank, sl].tobytes(), f"rank {rank}: worker error differs"
                if c.owner == rank:
                    assert et[sl].tobytes() == ost.et[sl].tobytes(), f"rank {rank}: server error differs"
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("comp", [Comp(SCALED_SIGN, use_ef=1), Comp(TOP_K, 1, 1000, use_ef=1),
                                  Comp(LINEAR_DITHER, bits=7, use_ef=0)], ids=["onebit", "topk", "ldither"])
def test_multi_rank_exchange_gloo(comp, world):
    import oracle
    oracle.build()
    from paper_2105_07829_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    comp_t = (comp.kind, comp.k_num, comp.k_den, comp.bits, comp.randk_scaled, comp.use_ef)
    procs = [ctx.Process(target=_worker, args=(r, world, port, comp_t, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res
