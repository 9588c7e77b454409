#!/usr/bin/env python
"""Summarise an ncu report (--page raw --csv) into key per-kernel metrics."""
import csv
import subprocess
import sys

KEYS = [
    ("time", "gpu__time_duration.sum", 1),
    ("dram_read", "dram__bytes_read.sum", 1),
    ("dram_write", "dram__bytes_write.sum", 1),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("dmma_inst_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("lsu_inst_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("shared_pipe_pct", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        print(f"== {r[ki][:90]}")
        for name, key, sc in KEYS:
            if key in h:
                v = r[h.index(key)].replace(",", "")
                try:
                    print(f"   {name:20s} {float(v) * sc:12.2f} {rows[1][h.index(key)]}")
                except ValueError:
                    print(f"   {name:20s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
