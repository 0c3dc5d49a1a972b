"""Summarise an ncu --csv launch list with NVLink counters (tools/gpu_r2_multi.sh):
per libbpc kernel launch, device, time, NVLink tx/rx user bytes, DRAM bytes."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    out = {}
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        k = (int(d["ID"]), d["Device"], d["Kernel Name"])
        out.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def main(path):
    rows = load(path)
    print("| id | dev | kernel | us | NVLink tx MB (user) | NVLink rx MB (user) | DRAM rd MB | DRAM wr MB |")
    print("|---|---|---|---|---|---|---|---|")
    for (i, dev, name), m in sorted(rows.items()):
        if "bpc::" not in name and "cstream" not in name and "update" not in name and "p2p" not in name:
            continue
        short = name.split("(")[0].replace("void ", "")
        print(f"| {i} | {dev} | {short} | {m.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
              f"{m.get('nvltx__bytes.sum', 0) / 1e6:.2f} ({m.get('nvltx__bytes_data_user.sum', 0) / 1e6:.2f}) | "
              f"{m.get('nvlrx__bytes.sum', 0) / 1e6:.2f} ({m.get('nvlrx__bytes_data_user.sum', 0) / 1e6:.2f}) | "
              f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
