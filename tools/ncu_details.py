#!/usr/bin/env python3
"""Print the headline metrics of an ncu report (details page) -- throughput, occupancy,
issue and warp-state figures -- for reading a --set full capture here.

  python tools/ncu_details.py report.ncu-rep [substring ...]
"""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Registers Per",
        "Theoretical Occupancy", "Issued Warp", "No Eligible", "Active Warps", "Eligible Warps",
        "L2 Hit", "L1/TEX Hit", "Block Limit", "Warp Cycles Per Issued", "SM Frequency", "Executed Ipc",
        "Stall", "Issue Slot", "L2 Cache Throughput", "L1/TEX Cache Throughput", "SM Busy", "Compute (SM)"]


def main():
    rep = sys.argv[1]
    keys = sys.argv[2:] or KEYS
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, si, ni, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    seen = set()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ni]
        if any(k in name for k in keys) and (r[si], name) not in seen:
            seen.add((r[si], name))
            print(f"{r[si]:40s} | {name:45s} | {r[ui]:10s} | {r[vi]}")


if __name__ == "__main__":
    main()
