"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes):
per kernel launches, ms/launch, GB/launch, share of the listed time; and the
per-phase DRAM bytes of the sweeps for profiles/ncu_traffic.json."""
import collections
import csv
import json
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    return per


def summary(path):
    per = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        name = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("sk::", "")
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':58s} {'n':>4s} {'ms/launch':>10s} {'GB/launch':>10s} {'share':>6s}"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n[:58]:58s} {c:4d} {t / c:10.4f} {b / c / 1e9:10.4f} {100 * t / tot:5.1f}%")
    return lines, agg


if __name__ == "__main__":
    lines, _ = summary(sys.argv[1])
    print("\n".join(lines))
