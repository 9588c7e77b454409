#!/usr/bin/env python
"""Per-kernel share of device time in an ncu --csv launch list (gpu__time_duration.sum).
Usage: python tools/launch_shares.py LAUNCHES.csv [LAST_N]  (LAST_N: only the last N launches)"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        launches[r[ii]] = (r[ki], float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0))
    items = list(launches.values())
    if len(sys.argv) > 2:
        items = items[-int(sys.argv[2]):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in items:
        agg[name[:90]][0] += 1
        agg[name[:90]][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(items)} launches, {tot / 1e3:.3f} ms total (ncu: cold caches, serialised)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:5d} {v[1]:11.1f} us {100 * v[1] / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
