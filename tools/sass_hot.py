"""Hot regions of an ncu source-page SASS export (csv, optionally .gz): per
kernel, instructions executed by opcode class and the top stall-sampled
instruction windows.  usage: sass_hot.py file.csv[.gz] [kernel-substring]"""
import csv
import gzip
import io
import re
import sys
from collections import Counter


def kernels(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        text = f.read()
    blocks = re.split(r'^"Kernel Name",', text, flags=re.M)
    for b in blocks[1:]:
        lines = b.split("\n", 1)
        name = lines[0].strip().strip(",").strip('"')
        rows = list(csv.reader(io.StringIO(lines[1])))
        yield name, rows[0], rows[1:]


def main(path, sub=""):
    for name, h, rows in kernels(path):
        if sub not in name:
            continue
        ix = {k: i for i, k in enumerate(h)}
        ops = Counter()
        stall = Counter()
        tot = 0
        samples = []
        for r in rows:
            if len(r) < len(h):
                continue
            src = r[ix["Source"]].strip()
            n = int(r[ix["Instructions Executed"]] or 0)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            opc = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
            ops[opc.split(".")[0]] += n
            stall[opc.split(".")[0]] += s
            tot += n
            samples.append((s, n, src))
        print(f"== {name[:90]}  warp-instructions {tot:,}")
        print("  by opcode (executed):", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(18)))
        st = sum(stall.values())
        print("  by opcode (stall samples):", ", ".join(f"{k} {v / st:.1%}" for k, v in stall.most_common(12)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")


def top_lines(path, sub="", n=40, ctx=3):
    for name, h, rows in kernels(path):
        if sub not in name:
            continue
        ix = {k: i for i, k in enumerate(h)}
        rows = [r for r in rows if len(r) >= len(h)]
        st = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows]
        tot = sum(st)
        order = sorted(range(len(rows)), key=lambda i: -st[i])[:n]
        for i in sorted(order):
            print(f"{i:6d} {st[i] / tot:6.2%} {int(rows[i][ix['Instructions Executed']] or 0):>11,}  {rows[i][ix['Source']].strip()[:90]}")
        return
