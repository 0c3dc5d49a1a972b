"""NVLink evidence for the fused exchange: n contexts of ONE process on n GPUs,
wired by bpc_connect_local (the same peer-memory kernels as the multi-process
transport), run a few steps of a config.  Meant to run under ncu with the
NVLink byte counters (tools/gpu_r2_multi.sh):

  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,... \
      python tools/nvlink_probe.py --config C5 --n 2

Every kernel launch of every device is listed with its NVLink transmit /
receive bytes, which tools/ncu_lines.py-style parsing compares with the
exchange's modeled volume (printed here as JSON: per rank, the bytes it pushes
to the other owners and the bytes of p it reads from them).  Plain run (no
ncu): also times the steps with CUDA events per device."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2105_07829_b200 as bpc
    from workloads import config, gen_grad_torch, gen_params

    n = args.n
    if torch.cuda.device_count() < n:
        raise SystemExit(f"needs {n} GPUs")
    w = config(args.config, n=n)
    streams, ctxs, xs, gs = [], [], [], []
    for r in range(n):
        dev = torch.device("cuda", r)
        with torch.cuda.device(r):
            s = torch.cuda.Stream(dev)
            streams.append(s)
            with torch.cuda.stream(s):
                ctxs.append(bpc.context_for(w, rank=r, world_size=n, device=r, stream=s.cuda_stream))
                xs.append(torch.tensor(gen_params(w), device=dev))
                gs.append(gen_grad_torch(w, r, 1, dev))
    for r in range(n):
        torch.cuda.synchronize(r)
    bpc.connect_local(ctxs)
    # modeled exchange bytes per rank and direction (payload segments of the other owners)
    model = []
    for r in range(n):
        seg = [ctxs[r].peer_segment(q)[1] for q in range(n)]
        model.append({"rank": r, "push_tx_bytes": sum(b for q, b in enumerate(seg) if q != r),
                      "pull_rx_bytes": sum(ctxs[q].peer_segment(q)[1] for q in range(n) if q != r)})
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n)]
    for it in range(args.steps):
        if it == args.steps - 1:
            for r in range(n):
                ev[r][0].record(streams[r])
        for r in range(n):
            ctxs[r].compress(gs[r])
        for c in ctxs:
            c.exchange_push()
        for c in ctxs:
            c.server()
        for c in ctxs:
            c.exchange_pull()
        for r in range(n):
            ctxs[r].step(xs[r], w.lr)
        if it == args.steps - 1:
            for r in range(n):
                ev[r][1].record(streams[r])
    for c in ctxs:
        c.sync()
    ms = [ev[r][0].elapsed_time(ev[r][1]) for r in range(n)]
    print(json.dumps({"config": args.config, "n": n, "exchange": ctxs[0].exchange,
                      "model": model, "last_step_ms_per_rank": ms}), flush=True)
    for c in ctxs:
        c.finalize()


if __name__ == "__main__":
    main()
