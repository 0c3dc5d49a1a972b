"""Where a kernel's issued instructions and stall samples go, from an ncu
source-page SASS export (`ncu -i r.ncu-rep --page source --csv --print-source sass`,
optionally gzipped): totals, the share spent in polling loops (the basic blocks
around NANOSLEEP / mbarrier try-waits), Philox multiplies, and stall reasons.
usage: ncu_source_breakdown.py file.csv[.gz]"""
import collections
import csv
import gzip
import io
import re
import sys


def kernels(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        text = f.read()
    seen = set()
    for b in re.split(r'^"Kernel Name",', text, flags=re.M)[1:]:
        name, rest = b.split("\n", 1)
        name = name.strip().strip(",").strip('"')
        if name in seen:
            continue
        seen.add(name)
        rows = list(csv.reader(io.StringIO(rest)))
        yield name, rows[0], [r for r in rows[1:] if len(r) > 5]


def poll_rows(src, cnt):
    """rows of the polling loops: the contiguous run of rows with the same executed
    count as a NANOSLEEP that executed more often than the instructions around it"""
    out = set()
    for i, s in enumerate(src):
        if "NANOSLEEP" not in s or cnt[i] == 0:
            continue
        c = cnt[i]
        lo = i
        while lo > 0 and cnt[lo - 1] == c:
            lo -= 1
        hi = i
        while hi + 1 < len(src) and cnt[hi + 1] == c:
            hi += 1
        out.update(range(lo, hi + 1))
    return out


def main(path):
    for name, h, rows in kernels(path):
        ix = {k: i for i, k in enumerate(h)}
        src = [r[ix["Source"]].strip() for r in rows]
        cnt = [int(r[ix["Instructions Executed"]] or 0) for r in rows]
        smp = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows]
        tot, stot = sum(cnt), sum(smp)
        poll = poll_rows(src, cnt)
        pin = sum(cnt[i] for i in poll)
        psm = sum(smp[i] for i in poll)
        phil = sum(c for s, c in zip(src, cnt) if "-0x2daee0ad" in s or "-0x326172a9" in s)
        reasons = collections.Counter()
        for r in rows:
            for k in h:
                if k.startswith("stall_") and "Not Issued" not in k:
                    reasons[k[6:]] += int(r[ix[k]] or 0)
        print(f"## `{name}`\n")
        print(f"* warp instructions executed: {tot:,}; stall samples: {stot:,}")
        print(f"* polling loops (mbarrier try-wait / nanosleep / counter spins): {pin / tot:.1%} of the "
              f"instructions, {psm / max(stot, 1):.1%} of the samples")
        print(f"* Philox multiplies (IMAD.WIDE / IMAD.HI by the round constants): {phil / tot:.1%} of the instructions")
        print("* stall samples by reason: " + ", ".join(f"{k} {v / stot:.1%}" for k, v in reasons.most_common(9)))
        print()


if __name__ == "__main__":
    main(sys.argv[1])
