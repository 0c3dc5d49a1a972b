"""Summaries for profiles/r2 from tools/gpu_r2_final.sh's output: per config a
markdown summary (the ncu launch list's per-kernel shares of the step, and the
--set full metrics of one step's kernels) and traffic.json (DRAM bytes per
launch of each kernel role, read by bench.py's roofline `traffic`).

usage: python tools/r2_summarize.py gpurun_out/final profiles/r2"""
import csv
import json
import os
import re
import sys
from collections import OrderedDict, defaultdict


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    per = OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if "Metric Name" not in d:
            continue
        key = (int(d["ID"]), d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return per


def short(name):
    name = name.replace("void ", "").replace("bpc::", "")
    return re.sub(r"\(.*\)$", "", name)


def role(name):
    n = short(name)
    m = re.match(r"cstream_kernel<(\d+), (\d+)", n)
    if m:
        return "server" if m.group(2) == "1" else "compress"
    if n.startswith("update_stream"):
        return "update"
    return None


def read_raw(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    units = dict(zip(h, rows[1]))
    return h, units, [dict(zip(h, r)) for r in rows[2:]]


def num(d, k):
    try:
        return float(str(d.get(k, "")).replace(",", ""))
    except ValueError:
        return None


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    traffic = {"_source": "ncu --set full --clock-control none of one step of `python bench.py --config <C> --steps 3 "
                          "--warmup 3 --no-e2e --no-cpu` (graph replay): dram__bytes_read.sum + "
                          "dram__bytes_write.sum per launch"}
    for cfg in ("C2", "C3", "C4", "C5"):
        out = [f"# {cfg}: ncu summary (round 2, HEAD)\n"]
        lp = os.path.join(src, f"launches_{cfg}.csv")
        if os.path.exists(lp):
            per = read_launches(lp)
            agg = defaultdict(lambda: [0, 0.0, 0.0])
            for (i, name), m in per.items():
                a = agg[short(name)]
                a[0] += 1
                a[1] += m.get("gpu__time_duration.sum", 0.0)
                a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            tot = sum(a[1] for a in agg.values())
            out.append("## Launch list (`--metrics gpu__time_duration.sum,dram__bytes_*` --clock-control none; "
                       "cold-cache, serialised: compare shares, not absolute times)\n")
            out.append("| kernel | launches | mean us | share of the listed time | DRAM MB / launch |")
            out.append("|---|---|---|---|---|")
            for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                unit_ns = 1e-3   # ncu reports nsecond for gpu__time_duration in csv mode
                out.append(f"| `{k}` | {c} | {t / c * unit_ns:.1f} | {t / tot:.1%} | {b / c / 1e6:.1f} |")
            out.append("")
        rp = os.path.join(src, f"full_{cfg}_raw.csv")
        if os.path.exists(rp):
            h, units, rows = read_raw(rp)
            out.append("## `--set full` (one step's kernels)\n")
            out.append("| kernel | us | DRAM GB | DRAM GB/s (of 6458.7 measured) | issue active % | warps active % | regs | "
                       "top stalls (per issue) |")
            out.append("|---|---|---|---|---|---|---|---|")
            stall_keys = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
                          k.endswith("_per_issue_active.ratio")]
            tr = defaultdict(list)
            for d in rows:
                name = d.get("Kernel Name", "")
                t = num(d, "gpu__time_duration.sum")
                tu = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
                if t is not None:
                    t *= tu.get(units.get("gpu__time_duration.sum", "us"), 1.0)   # -> microseconds
                rb = num(d, "dram__bytes_read.sum") or 0.0
                wb = num(d, "dram__bytes_write.sum") or 0.0
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rb *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
                wb *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
                st = sorted(((num(d, k) or 0.0, k) for k in stall_keys), reverse=True)[:3]
                sts = ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
                                f"{v:.2f}" for v, k in st)
                gbs = (rb + wb) / (t * 1e-6) / 1e9 if t else 0.0
                out.append(f"| `{short(name)}` | {t:.1f} | {(rb + wb) / 1e9:.3f} | {gbs:.0f} ({gbs / 6458.7:.2f}) | "
                           f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0:.1f} | "
                           f"{num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0:.1f} | "
                           f"{d.get('launch__registers_per_thread', '')} | {sts} |")
                r = role(name)
                if r:
                    tr[r].append(rb + wb)
            traffic[cfg] = {r: int(sum(v) / len(v)) for r, v in tr.items()}
            out.append("")
        with open(os.path.join(dst, f"{cfg}_summary.md"), "w") as f:
            f.write("\n".join(out) + "\n")
    with open(os.path.join(dst, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
