"""Automatic size-threshold search (PAPER.md:504-505:
"We leave the automatic threshold search as future work. Currently, we set the
threshold to 1MB by default").

For each candidate threshold th (tensors with 4 * numel < th stay raw fp32,
DESIGN.md R3) the tool
  1. runs `bench.py --threshold-bytes th` on this GPU and reads the measured
     device step time t_dev(th) (CUDA events, N=1) and the payload P(th) that
     libbpc's chunk plan produces per rank and direction;
  2. models the step on an n-rank job whose exchange runs over a link of
     `link_gbs` GB/s per direction: push then pull (Alg. 4 l.6-12),
     each moving P * (n - 1) / n bytes per GPU (Table 1):
         T(th) = t_dev(th) + 2 * P(th) * (n - 1) / n / link_bw
and picks the threshold with the smallest T. The device time is measured, the
communication term is a model (NVLink / NVSwitch: 900 GB/s; the paper's
25 Gb/s Ethernet: 3.125 GB/s), so the choice shows how the best threshold moves
with the network the job runs on.

Usage (on a GPU box):
  python tools/threshold_search.py --config C2 [--n 8] [--link-gbs 900 3.125] [--steps 200]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [0, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24]


def modeled_ms(t_dev_ms: float, payload_bytes: int, n: int, link_gbs: float) -> float:
    """T(th) of the module docstring, in ms."""
    return t_dev_ms + 2.0 * payload_bytes * (n - 1) / n / (link_gbs * 1e9) * 1e3


def choose(rows: list[dict], n: int, link_gbs: float) -> dict:
    """The row (threshold_bytes, ms_per_step, payload_bytes) with the smallest
    modeled step time; ties go to the larger threshold (fewer compressed units)."""
    return min(rows, key=lambda r: (modeled_ms(r["ms_per_step"], r["payload_bytes"], n, link_gbs),
                                    -r["threshold_bytes"]))


def measure(cfg: str, th: int, steps: int, warmup: int) -> dict:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--threshold-bytes", str(th),
           "--steps", str(steps), "--warmup", str(warmup), "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    if r.returncode != 0:
        raise RuntimeError(f"bench.py failed at threshold {th}: {r.stderr[-1500:]}")
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    return {"threshold_bytes": th, "ms_per_step": line["ms_per_step"],
            "payload_bytes": line["config"]["payload_bytes_per_rank"],
            "compressed_chunks": line["config"]["compressed_chunks"], "chunks": line["config"]["chunks"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=8, help="ranks of the modeled job")
    ap.add_argument("--link-gbs", type=float, nargs="+", default=[900.0, 3.125])
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    rows = [measure(a.config, th, a.steps, a.warmup) for th in CANDIDATES]
    out = {"config": a.config, "n_modeled": a.n, "rows": rows, "best": {}}
    for bw in a.link_gbs:
        b = choose(rows, a.n, bw)
        out["best"][str(bw)] = {"threshold_bytes": b["threshold_bytes"],
                                "modeled_ms": round(modeled_ms(b["ms_per_step"], b["payload_bytes"], a.n, bw), 5)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
