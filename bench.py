#!/usr/bin/env python
"""bench.py — the compressed aggregate + update step of arXiv 2105.07829 on B200.

One step = one pass of the whole hot path over one
synthetic gradient per rank: bpc_compress (worker EF + compression) ->
bpc_aggregate (all-to-all of payloads, server decompress-sum-recompress,
all-gather; over NVLink peer memory fused into the kernels, or NCCL with
--exchange nccl) -> bpc_step (fused decode + Adam).

Metric (BASELINE.json): gradient GB/s = (ranks x 4 bytes x d) / step time,
d = the model's parameter count; whole-job aggregate over all ranks.

Launch: python bench.py [--config C2] [--steps K] [--warmup W]
        torchrun --nproc-per-node N bench.py --gpus N ...
        python bench.py --impl reference   (the CPU oracle, timed on host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed aggregate+update step: gradient GB/s per step at 1/2/4/8 B200, % roofline"
DESCR = {
    "C1": "d=4096 synthetic gradient, onebit scaled-sign + EF (configs[0])",
    "C2": "ResNet-50-shaped gradient (25.6M params, 161 tensors), onebit two-way + EF + Adam (configs[1])",
    "C3": "VGG16-shaped gradient (138M params), top-k 0.1% (binary16 values, PAPER.md:648) + EF + Adam (configs[2])",
    "C4": "BERT-base-shaped gradient (110M params), linear dithering 7 bits (Alg. 3) + Adam (configs[3])",
    "C5": "BERT-large-shaped gradient (336M params), onebit two-way + EF + Adam (configs[4])",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5",
                    help="workload (BASELINE.json configs): C5 BERT-large = the largest single-GPU config, the "
                         "metric's default; C2 ResNet-50, C3 VGG16, C4 BERT-base, C1 d=4096")
    ap.add_argument("--exchange", choices=["auto", "p2p", "nccl", "nvls"], default="auto",
                    help="N>1 transport of the push/pull exchange: NVLink peer stores, NCCL send/recv, or "
                         "peer stores + an NVLS multicast pull; auto = nvls for scaled sign with raw units "
                         "< 25%% of the payload (measured faster: C5), else p2p")
    ap.add_argument("--optimizer", choices=["adam", "lans", "nag"], default="adam",
                    help="bpc_step update: Adam core (A9), the LANS / CLAN block-normalised update (NEXT #1) "
                         "or NAG (the CNN runs' optimizer, R24)")
    ap.add_argument("--units", choices=["chunk", "tensor"], default="chunk",
                    help="compression unit: 2^18-element chunks (R1) or whole tensors (PAPER.md:505; norm "
                         "kinds: two-pass kernels, sparse kinds: the large-unit select path)")
    ap.add_argument("--threshold-bytes", type=int, default=None,
                    help="size threshold (PAPER.md:504-505): tensors below it stay raw; default: the config's 1 MiB "
                         "(tools/threshold_search.py sweeps it)")
    ap.add_argument("--launch", choices=["graph", "eager"], default="graph",
                    help="timed steps: replay of a CUDA graph of one whole step (default; t and the "
                         "exchange epochs advance on the device) or eager calls")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU work per cpu_baseline leg (1 core, then all host cores)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler running around the timed region (B200_PROFILING.md)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self, t0=None, t1=None):
        """Median SM clock and throttle reasons over the samples inside [t0, t1]
        (host wall clock of the timed region); all samples if none fall inside."""
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        import datetime
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]),
                             [nm for nm, v in zip(names, parts[3:7]) if v.lower() == "active"]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        win = [r for r in rows if t0 is not None and t0 - 0.06 <= r[0] <= t1 + 0.06]
        scope = "timed region"
        if not win:
            win, scope = rows, "whole run (no sample fell inside the timed region)"
        sm = sorted(r[1] for r in win)
        reasons = sorted({x for r in win for x in r[3]})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max((r[2] for r in win), default=None),
                "reasons": reasons, "samples": len(win), "window": scope}


# ---------------------------------------------------------------- byte models
def kernel_bytes(chunks, comp, n, rank, lans=False, nag=False, per_tensor=False):
    """Algorithmic HBM bytes per launch of each kernel; LANS's
    update = pass 1 (m, v, x read, m, v written) + pass 2 (m, v, x read, x
    written) + the payload read twice; per-tensor units read the worker's
    g, e (server: e~ and the payloads) once more in their first pass."""
    ef = comp.use_ef
    sparse = comp.kind in (3, 4)
    w = s = u = 0
    for c in chunks:
        L, pb = c.len, c.payload_bytes
        if c.raw:
            w += 8 * L
            if c.owner == rank:
                s += 4 * n * L + 4 * L
            u += (36 * L + 8 * L) if lans else (16 * L + 4 * L) if nag else (24 * L + 4 * L)
        elif sparse:
            # worker: g, e read, e written; server: Delta read (e~ is written only at
            # the k selected and the ranks' entries); units > 2^18 (per-tensor) read
            # q / Delta twice more (slice counts, ordered emission)
            big = 8 * L if L > (1 << 18) else 0
            w += (12 if ef else 4) * L + pb + big
            if c.owner == rank:
                s += n * pb + 4 * L + pb + big
            u += (36 * L + 2 * pb) if lans else (16 * L + pb) if nag else (24 * L + pb)
        else:
            w += (12 if ef else 4) * L + pb + ((8 if ef else 4) * L if per_tensor else 0)
            if c.owner == rank:
                s += n * pb + (8 * L if ef else 0) + pb + ((4 * L if ef else 0) + n * pb if per_tensor else 0)
            u += (36 * L + 2 * pb) if lans else (16 * L + pb) if nag else (24 * L + pb)
    return {"compress": w, "server": s, "update": u}


def ncu_traffic(cfg_name, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    of the same workload (profiles/*/traffic.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                v = json.load(f).get(cfg_name, {}).get(kernel)
            if v:
                return int(v), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- CPU oracle leg
def host_cpu():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def oracle_sample(wcfg, n, seconds, threads):
    """Time the oracle as it stands on `threads` host cores (OpenMP over units,
    bit-identical to 1 thread) on a bounded sample of the workload: the config
    with every tensor, the size threshold and the unit size divided by s (tensor
    count and raw / compressed mix kept), s chosen for ~seconds/3 per round,
    rounds repeated until `seconds` of wall time; gradient GB/s = n x 4 d_sample / s."""
    import numpy as np

    import oracle
    from workloads import gen_grad, gen_params, layout
    oracle.build()
    d_full = sum(wcfg.tensor_numels())
    rate = 12e6 * threads / max(1, n)              # oracle elements / s (measured ~15e6 per core, n = 1)
    s = max(1, int(np.ceil(d_full / (rate * seconds / 3))))
    w = wcfg if s == 1 else replace(wcfg, scale=s, threshold_bytes=wcfg.threshold_bytes // s,
                                     chunk_elems=max(1, wcfg.chunk_elems // s) if wcfg.chunk_elems else 0)
    numels = w.tensor_numels()
    offs, D = layout(numels)
    d = sum(numels)
    cfg = oracle.Cfg.from_workload(w, n=n)
    st = oracle.State(n, D, gen_params(w))
    grads = [np.stack([gen_grad(w, i, k) for i in range(n)]) for k in (1, 2)]
    oracle.set_threads(threads)
    steps, busy = 0, 0.0
    try:
        while busy < seconds or steps == 0:
            t0 = time.perf_counter()
            oracle.round_(cfg, st, grads[steps % 2], w.lr, want_payloads=False)
            busy += time.perf_counter() - t0
            steps += 1
    finally:
        oracle.set_threads(1)
    return n * 4 * d * steps / busy / 1e9, steps, busy, s, d


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle
    from workloads import config, gen_grad, gen_params, layout
    n = args.gpus
    full = config(args.config, n=n,
                  **({"threshold_bytes": args.threshold_bytes} if args.threshold_bytes is not None else {}))
    d_full = sum(full.tensor_numels())
    # Each step is one oracle round (n simulated workers) over a miniature of the
    # workload: every tensor, the size threshold and the unit size divided by s,
    # so the tensor count and the raw / compressed mix are kept; s is chosen so
    # the whole --warmup + --steps run takes about a minute on one core.
    rate = 12e6 * host_cpu()[1]                    # oracle elements / s on all cores (~15e6 per core)
    budget = max(4096.0, 60.0 * rate / max(1, args.steps + args.warmup) / n)
    s = max(1, int(np.ceil(d_full / budget)))
    w = config(args.config, n=n, scale=s, threshold_bytes=full.threshold_bytes // s,
               chunk_elems=max(1, full.chunk_elems // s), optimizer=args.optimizer)
    oracle.build()
    numels = w.tensor_numels()
    offs, D = layout(numels)
    d = sum(numels)
    cfg = oracle.Cfg.from_workload(w, n=n)
    st = oracle.State(n, D, gen_params(w))
    grads = [np.stack([gen_grad(w, i, k) for i in range(n)]) for k in (1, 2)]
    model, ncores = host_cpu()
    oracle.set_threads(ncores)               # the oracle on all host cores (OpenMP over units)
    for i in range(args.warmup):
        oracle.round_(cfg, st, grads[i % 2], w.lr, want_payloads=False)
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.round_(cfg, st, grads[i % 2], w.lr, want_payloads=False)
    busy = time.perf_counter() - t0
    steps = args.steps
    ms = busy / steps * 1e3
    val = n * 4 * d * steps / busy / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {DESCR[args.config]}", "ranks_simulated": n, "d": d_full,
                   "sample_scale": s, "sample_d": d},
        "cpu_baseline": {"value": round(val, 6), "unit": "GB/s", "cores": ncores, "kind": "oracle",
                         "cpu_model": model,
                         "sample": f"each step: one oracle round of {args.config} with every tensor, the threshold "
                                   f"and the unit size divided by {s} ({d} elements), {n} simulated workers, "
                                   f"OpenMP over units on {ncores} host cores"},
        "e2e": {"value": round(val, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    clocks = Clocks(local)   # started early: nvidia-smi needs ~0.5 s before its first sample
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2105_07829_b200 import build as bbuild
    if rank == 0 and not os.path.exists(bbuild.LIB):
        bbuild.build()
    if world > 1:
        dist.barrier()
    import paper_2105_07829_b200 as bpc
    from workloads import config, gen_grad_torch, gen_params, layout

    w = config(args.config, n=world, optimizer=args.optimizer,
               **({"chunk_elems": 0} if args.units == "tensor" else {}),
               **({"threshold_bytes": args.threshold_bytes} if args.threshold_bytes is not None else {}))
    numels = w.tensor_numels()
    offs, D = layout(numels)
    d = sum(numels)
    nid = None
    if world > 1:
        obj = [bpc.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    exchange = args.exchange
    if exchange == "auto":
        # measured at N = 2 / 4: the multicast pull wins where the
        # payload is sign bits (coalesced 4-byte multimem stores); raw-heavy (C2)
        # and dithering payloads (strided code words) lose
        if world > 1 and w.comp.kind == 2:
            s_, chs = bpc.plan(bpc.make_config(numels, offs, w.comp, world_size=world,
                                               chunk_elems=w.chunk_elems or (1 << 18),
                                               threshold_bytes=w.threshold_bytes))
            raw = sum(c.payload_bytes for c in chs if c.raw)
            exchange = "nvls" if raw < 0.25 * max(1, s_.payload_total) else "p2p"
        else:
            exchange = "p2p"
    stream = torch.cuda.Stream(dev)   # a capturable stream (not the legacy default stream)
    torch.cuda.set_stream(stream)
    ctx = bpc.context_for(w, rank=rank, world_size=world, device=local, stream=stream.cuda_stream, nccl_id=nid,
                          exchange=exchange)
    chunks = ctx.chunks()
    grads = [gen_grad_torch(w, rank, s, dev) for s in (1, 2)]
    x = torch.tensor(gen_params(w), device=dev)
    torch.cuda.synchronize()

    def step(i):
        ctx.compress(grads[i % 2])
        ctx.aggregate()
        ctx.step(x, w.lr)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        step(i)
    barrier()
    run = step
    if args.launch == "graph":
        # one CUDA graph per gradient buffer, each one whole step (compress, push,
        # server, pull, update); every replay is the next step (device-side t / epochs)
        graphs, per_graph = [], []
        for b in (0, 1):
            graphs.append(torch.cuda.CUDAGraph())
            l0 = ctx.launch_count()
            with torch.cuda.graph(graphs[-1], stream=stream):
                step(b)
            per_graph.append(ctx.launch_count() - l0)
        barrier()
        for i in range(2):   # first replays (graph upload) stay out of the timed region
            graphs[i].replay()
        barrier()
        run = lambda i: graphs[i % 2].replay()
    launches0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wt0 = time.time()
    e0.record(stream)
    for i in range(args.steps):
        run(i)
    e1.record(stream)
    barrier()
    wt1 = time.time()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = ctx.launch_count() - launches0
    if args.launch == "graph":
        launches = sum(per_graph[i % 2] for i in range(args.steps))
    clk = clocks.stop(wt0, wt1)
    ctx.sync()

    # per-kernel device timing (events recorded by libbpc around each launch, same stream)
    # (eager launches with two events per phase; bounded: thousands of live
    # events make cudaEventCreate slow enough to leave the GPU waiting)
    ctx.set_timing(True)
    for i in range(min(args.steps, 200)):
        step(i)
    barrier()
    tim = ctx.timing()
    ctx.set_timing(False)
    kb = kernel_bytes(chunks, w.comp, world, rank, lans=args.optimizer == "lans", nag=args.optimizer == "nag",
                      per_tensor=args.units == "tensor")
    per = {k: (tim[k][0] / max(1, tim[k][1]), tim[k][1]) for k in ("compress", "server", "update", "push", "pull")}
    dom = max(("compress", "server", "update"), key=lambda k: per[k][0])
    peak, peak_src = peaks()
    achieved = kb[dom] / (per[dom][0] * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.config, dom) if world == 1 else (None, None)
    kern = {k: {"ms": round(per[k][0], 5), "GB/s": round(kb[k] / max(per[k][0], 1e-9) / 1e6, 1) if k in kb else None,
                "frac": round(kb[k] / max(per[k][0], 1e-9) / 1e6 / peak, 4) if k in kb else None,
                "alg_bytes": kb.get(k)} for k in per if per[k][1]}
    # step roofline: t_roof = max(sum of the kernels' algorithmic HBM
    # bytes / HBM peak, exchange bytes per direction / 900 GB/s) against the step time
    step_bytes = sum(kb.values())
    nvl_bytes = 0
    if world > 1:
        nvl_bytes = sum(ctx.peer_segment(r)[1] for r in range(world) if r != rank)   # per direction, push or pull
    t_roof = max(step_bytes / (peak * 1e9), 2 * nvl_bytes / 900e9 if world > 1 else 0.0)
    t_roof8 = max(step_bytes / 8000e9, 2 * nvl_bytes / 900e9 if world > 1 else 0.0)

    # end to end through the public API: pinned host gradient -> device, step, params -> host
    e2e = None
    if not args.no_e2e:
        # End to end through the public API with HOST buffers, pipelined the way a
        # data loader would run it: step i's gradient is copied host->device on
        # an H2D stream (double-buffered), the step runs on the compute stream,
        # and its result x is snapshotted on the device and read back to pinned
        # host memory on a D2H stream, so the two PCIe directions and the compute
        # overlap across steps.  Every step's copies are inside the timed region.
        hg = [grads[s].cpu().pin_memory() for s in (0, 1)]
        hx = [torch.empty(x.shape, dtype=torch.float32).pin_memory() for _ in (0, 1)]
        dg = [torch.empty_like(grads[0]) for _ in (0, 1)]
        xs = [torch.empty_like(x) for _ in (0, 1)]
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()
        g_ready = [ev(), ev()]
        g_free = [ev(), ev()]
        x_snap = [ev(), ev()]
        x_read = [ev(), ev()]
        for b in (0, 1):
            g_free[b].record(stream)
            x_read[b].record(stream)

        def e2e_step(i):
            b = i % 2
            with torch.cuda.stream(s_h2d):
                s_h2d.wait_event(g_free[b])
                dg[b].copy_(hg[b], non_blocking=True)
                g_ready[b].record(s_h2d)
            stream.wait_event(g_ready[b])
            ctx.compress(dg[b])
            g_free[b].record(stream)
            ctx.aggregate()
            ctx.step(x, w.lr)
            stream.wait_event(x_read[b])
            xs[b].copy_(x, non_blocking=True)
            x_snap[b].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(x_snap[b])
                hx[b].copy_(xs[b], non_blocking=True)
                x_read[b].record(s_d2h)

        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize()
        barrier()
        k2 = max(2, min(args.steps, 50))
        e0.record(stream)
        for i in range(k2):
            e2e_step(i)
        stream.wait_stream(s_d2h)
        e1.record(stream)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / k2)
        e2e = {"value": round(world * 4 * d / (ms_e2e * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": 4 * D, "d2h_bytes_per_step": 4 * D, "ms_per_step": round(ms_e2e, 4),
               "note": "pinned host g -> device (H2D stream, double-buffered), step, x -> pinned host "
                       "(device snapshot + D2H stream); copies overlap compute across steps"}
    ctx.sync()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        model, ncores = host_cpu()
        legs = {}
        for th in sorted({1, ncores}):
            val, steps, busy, sc, ds = oracle_sample(w, 1, args.cpu_seconds, th)
            legs[th] = {"value": round(val, 6), "unit": "GB/s", "cores": th,
                        "sample": f"{steps} oracle rounds of {args.config} with every tensor, the threshold and "
                                  f"the unit size divided by {sc} ({ds} elements, n=1), {busy:.1f} s on {th} "
                                  f"host core(s)"}
        cpu = dict(legs[ncores], kind="oracle", cpu_model=model, nproc=ncores, single_core=legs[1])

    if rank == 0:
        s = ctx.summary()
        line = {
            "metric": METRIC, "value": round(world * 4 * d / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {DESCR[args.config]}", "d": d, "tensors": len(numels),
                       "chunks": s.num_chunks, "compressed_chunks": s.num_compressed,
                       "payload_bytes_per_rank": s.payload_total,
                       "compression_rate_vs_fp32": round(4 * d / s.payload_total, 2),
                       "l2": "inputs larger than L2 (g, e, m, v, x = %.0f MB per rank)" % (20 * D / 1e6),
                       "parallelism": f"dp{world} (sharded server: all-to-all + all-gather)",
                       "exchange": ctx.exchange if world > 1 else None,
                       "optimizer": args.optimizer, "units": args.units, "launch": args.launch,
                       "threshold_bytes": w.threshold_bytes},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "alg_bytes_per_launch": kb[dom],
                         "step_bytes": step_bytes, "step_frac": round(t_roof * 1e3 / ms, 4),
                         "step_frac_8tbs": round(t_roof8 * 1e3 / ms, 4),
                         "step_note": "step_frac = max(sum of algorithmic HBM bytes of the step / peak, "
                                      "exchange bytes / 900 GB/s) / ms_per_step; step_frac_8tbs uses the north "
                                      "star's 8 TB/s"},
            "kernels": kern,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world > 1:
            # NVLink traffic of the exchange, per GPU and direction: the worker sends
            # the other owners' segments (push), the update reads the other owners'
            # p (pull); averaged over the step it is a small fraction of 900 GB/s
            seg = [ctx.peer_segment(r)[1] for r in range(world)]
            per_dir = sum(b for r, b in enumerate(seg) if r != rank)
            line["nvlink"] = {"bytes_per_step_per_direction": per_dir,
                              "avg_GBps_per_direction": round(per_dir / (ms * 1e-3) / 1e9, 3),
                              "peak_GBps_per_direction": 900.0,
                              "source": "payload bytes of the other owners' segments (plan), not a counter; "
                                        "ncu NVLink counters: profiles/r2/nvlink_*"}
            # bus bandwidth per nccl-tests: the bytes a rank receives, P (n - 1) / n, over
            # the exchange's own time; only where the exchange is its own launch (NCCL,
            # or the sparse kinds' copy kernels) - the fused exchange has no such time
            bus = {}
            for k in ("push", "pull"):
                if per[k][1]:
                    bus[k + "_ms"] = round(per[k][0], 5)
                    bus[k + "_busbw_GBps"] = round(per_dir / (per[k][0] * 1e-3) / 1e9, 2)
            if bus:
                line["bus"] = bus
        print(json.dumps(line), flush=True)
    # the graphs hold the captured launches (NCCL kernels included): release them
    # before the context's communicator and buffers go
    run = graphs = None
    torch.cuda.synchronize()
    ctx.finalize()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
