#!/usr/bin/env python
"""Print selected raw ncu metrics per kernel launch (dev tool).

Usage: python tools/ncu_metrics.py REPORT.ncu-rep [REGEX ...]
Default regexes: duration, tensor-pipe activity, smem wavefronts, issue activity, DRAM bytes,
warp stall reasons.
"""
import csv
import io
import re
import subprocess
import sys

DEFAULT = [r"^gpu__time_duration.sum$", r"pipe_tensor_cycles_active_realtime.*pct_of_peak_sustained_elapsed",
           r"^sm__pipe_tensor_subpipe_hmma_cycles_active_realtime", r"data_pipe_tc_wavefronts_mem_shared.sum.pct",
           r"^smsp__issue_active.avg.pct", r"^dram__bytes_(read|write).sum$", r"pipe_tmem.avg.pct",
           r"smsp__average_warp_latency_issue_stalled_.*\.ratio$|smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$"]


def main():
    rep = sys.argv[1]
    pats = [re.compile(p) for p in (sys.argv[2:] or DEFAULT)]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        print("==", r[ki][:90])
        for i, h in enumerate(hdr):
            if any(p.search(h) for p in pats):
                v = r[i]
                try:
                    if float(v.replace(",", "")) == 0.0 and "stalled" in h:
                        continue
                except ValueError:
                    pass
                print(f"   {h[:95]:95s} {v:>14s} {units[i]}")


if __name__ == "__main__":
    main()
