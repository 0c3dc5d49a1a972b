"""Per-source-line instruction and stall-sample shares of one kernel of an
ncu report (`ncu -i REP --page source --print-source cuda,sass --csv`).
usage: python tools/ncu_lines.py REP [launch_index] [top]"""
import csv
import io
import subprocess
import sys


def lines(rep, idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    res, f = [], None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or len(r) < 8:
            continue
        if r[0]:   # a source line row (aggregated over its SASS)
            try:
                res.append((f, int(r[0]), r[1].strip(), int(r[7].replace(",", "")), int(r[4].replace(",", ""))))
            except ValueError:
                pass
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    L = lines(rep, idx)
    ti = sum(x[3] for x in L) or 1
    ts = sum(x[4] for x in L) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for f, n, src, ins, st in sorted(L, key=lambda x: -x[3])[:top]:
        print(f"{ins / ti * 100:5.1f}% inst {st / ts * 100:5.1f}% stall  {f}:{n}  {src[:90]}")
