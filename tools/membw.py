#!/usr/bin/env python
"""Per-kernel DRAM bandwidth from an ncu launch list with dram__bytes_read/write and
gpu__time_duration (the memory-roofline view of the memory-bound passes).
Usage: python tools/membw.py LAUNCHES.csv [PEAK_GBPS]"""
import collections
import csv
import sys

SCALE_T = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6550.0
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H = rows[h]
    ki, mi, vi, ui, ii = (H.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    d = collections.defaultdict(dict)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        sc = SCALE_T.get(r[ui]) or SCALE_B.get(r[ui]) or 1.0
        d[r[ii]]["name"] = r[ki]
        d[r[ii]][r[mi]] = v * sc
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for v in d.values():
        nm = v["name"].split("(")[0].replace("void ", "").replace("nmg::<unnamed>::", "")[:40]
        a = agg[nm]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':42s} {'n':>4s} {'time ms':>9s} {'share':>6s} {'GB/s':>8s} {'of peak':>7s}")
    for nm, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        bw = b / t / 1e9 if t else 0.0
        print(f"{nm:42s} {n:4d} {t * 1e3:9.3f} {100 * t / tot:5.1f}% {bw:8.0f} {100 * bw / peak:6.1f}%")


if __name__ == "__main__":
    main()
