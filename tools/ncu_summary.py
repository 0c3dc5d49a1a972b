"""Summarise ncu output for profiles/: a launch list CSV (per-launch device time,
DRAM bytes) and/or a `--set full` report (.ncu-rep, read with `ncu -i`).

usage: python tools/ncu_summary.py [--launches gpurun_out/launches.csv] [--rep gpurun_out/prof.ncu-rep]
                                   [--traffic CFG --out profiles/<round>/traffic.json]
--traffic merges the report's per-launch DRAM bytes (read + write), averaged per
kernel role (compress / server / update), into the traffic JSON under CFG.
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__inst_executed.avg.per_cycle_active", "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__average_warps_issue_stalled_barrier_per_issue_active",
]


def short(name: str) -> str:
    for k in ("compress_kernel<2, false>", "compress_kernel<2, true>"):
        pass
    name = name.replace("void bpc::", "").replace("(bpc::CompressParams)", "").replace("(bpc::UpdateParams)", "")
    return name.strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        names[r[idi]] = short(r[ki])
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if unit in ("nsecond", "ns"):
            v /= 1e3
        elif unit in ("msecond", "ms"):
            v *= 1e3
        elif unit in ("usecond", "us"):
            pass
        elif unit in ("byte",):
            pass
        elif unit == "Kbyte":
            v *= 1e3
        elif unit == "Mbyte":
            v *= 1e6
        elif unit == "Gbyte":
            v *= 1e9
        per[r[idi]][r[mi]] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i]]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    out = ["| kernel | launches | mean us | share | DRAM MB/launch | DRAM GB/s |", "|---|---|---|---|---|---|"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{n}` | {c} | {t / c:.1f} | {t / tot:.1%} | {b / c / 1e6:.1f} | {b / (t * 1e-6) / 1e9 if t else 0:.0f} |")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        name = short(r[col["Kernel Name"]])
        out.append(f"### `{name}`")
        for m in METRICS:
            if m in col:
                out.append(f"- {m}: {r[col[m]]} {units[col[m]]}")
        stalls = [(h, r[i]) for h, i in col.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and r[i]]
        top = sorted(((h, float(v.replace(",", ""))) for h, v in stalls if v.replace(",", "").replace(".", "").isdigit()),
                     key=lambda x: -x[1])[:6]
        if top:
            out.append("- top stall samples: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v:.0f}" for h, v in top))
    return "\n".join(out)


def role(name: str):
    if "update" in name:
        return "update"
    for pat, r in (("stream_kernel<", None), ("compress_kernel<", None)):
        if pat in name:
            args = name.split(pat, 1)[1].split(">", 1)[0].replace("(int)", "").replace("(bool)", "")
            parts = [a.strip() for a in args.split(",")]
            server = parts[1] in ("1", "true")
            return "server" if server else "compress"
    return None


def traffic(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = defaultdict(list)
    for r in rows[2:]:
        rl = role(r[col["Kernel Name"]])
        if rl is None:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[m]].replace(",", "")) * scale[units[col[m]]]
        acc[rl].append(b)
    return {k: int(sum(v) / len(v)) for k, v in acc.items()}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--traffic")
    ap.add_argument("--out")
    a = ap.parse_args()
    if a.traffic:
        import json
        import os
        d = json.load(open(a.out)) if a.out and os.path.exists(a.out) else {}
        d["_source"] = ("ncu --set full --clock-control none captures of `python bench.py --config <C> --steps 5 "
                        "--warmup 3 --no-e2e --no-cpu`: dram__bytes_read.sum + dram__bytes_write.sum per launch")
        d[a.traffic] = traffic(a.rep)
        json.dump(d, open(a.out, "w"), indent=1)
        print(a.traffic, d[a.traffic])
        raise SystemExit
    if a.launches:
        print(launches(a.launches))
    if a.rep:
        print(report(a.rep))
