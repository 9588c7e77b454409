#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples / executed instructions per kernel (dev tool).

Usage: ncu -i R.ncu-rep --page source --csv --print-source sass > s.csv
       python tools/ncu_sass_top.py s.csv [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1]
            hdr = rows[i + 1]
            j = i + 2
            body = []
            while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
                body.append(rows[j])
                j += 1
            si, ni, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
                "Warp Stall Sampling (Not-issued Samples)"), hdr.index("Instructions Executed")
            tot = sum(int(r[si] or 0) for r in body)
            tote = sum(int(r[ei] or 0) for r in body)
            print(f"== {name[:100]}  samples {tot}  warp-instr {tote}")
            body_idx = list(enumerate(body))
            for k, r in sorted(body_idx, key=lambda x: -int(x[1][si] or 0))[:top]:
                print(f"  {k:5d} {int(r[si] or 0):7d} {int(r[ni] or 0):7d} {int(r[ei] or 0):9d}  {r[1].strip()[:80]}")
            i = j
        else:
            i += 1


if __name__ == "__main__":
    main()
