#!/usr/bin/env python
"""Aggregate an ncu CSV (metrics dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum)
of `bench.py --steps 1` into per-kernel-class DRAM bytes of ONE step (the last `per_step` launches of
the library, PER_STEP = the bench line's real kernel count per step, sum of launches_per_step) and
merge them into profiles/traffic.json under the key KEY (e.g. "cfg1").
Usage: ncu_traffic.py CSV PER_STEP_LAUNCHES OUT KEY"""
import collections
import csv
import json
import sys

# the library's kernel classes (include/nmg.h NMG_K_*): first match wins
CLASS = [("dgemm", "gemm64"), ("ozaki", "gemm64"), ("row_sumsq", "misc"), ("row_norms", "misc"),
         ("tc_gemm", "gemm32"), ("kron_tc", "gemm32"), ("sgemm", "gemm32"), ("gemm_f32", "gemm32"),
         ("smooth1d", "smooth"), ("strip_combine", "filter"), ("conv_strip", "smooth"), ("cycle64", "smooth"),
         ("fno_", "smooth"), ("cnn2d", "smooth"), ("combine_rows_fft", "filter"), ("fft_", "filter"),
         ("sumsq", "filter"), ("real_to_complex", "filter"),
         ("restrict", "transfer"), ("prolong", "transfer"), ("coarse", "coarse")]


def cls(name):
    for key, c in CLASS:
        if key in name:
            return c
    return "misc"


def main(path, per_step, out, key):
    rows = list(csv.reader(open(path)))
    h = [r for r in rows if "Kernel Name" in r][0]
    hi = rows.index(h)
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or "nmg::" not in r[ki]:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
                 "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1)
        launches.setdefault(r[ii], {"name": r[ki]})[r[mi]] = v * scale
    last = list(launches.values())[-per_step:]
    agg = collections.defaultdict(lambda: {"bytes": 0.0, "s": 0.0, "n": 0})
    for L in last:
        c = agg[cls(L["name"])]
        c["bytes"] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
        c["s"] += L.get("gpu__time_duration.sum", 0)
        c["n"] += 1
    res = {k: v["bytes"] for k, v in agg.items()}
    try:
        allres = json.load(open(out))
    except Exception:
        allres = {}
    if not all(isinstance(v, dict) for v in allres.values()):
        allres = {}
    allres[key] = res
    json.dump(allres, open(out, "w"), indent=1)
    for k, v in agg.items():
        print(f"{k:9s} launches {v['n']:3d}  dram {v['bytes'] / 1e6:10.1f} MB  time {v['s'] * 1e3:8.3f} ms (cold, serialised)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4])
