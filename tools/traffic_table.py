#!/usr/bin/env python3
"""gpurun_out/tr_<kernel>_<cfg>_p<p>.csv (tools/profile_traffic_v3.sh) -> markdown table of
DRAM bytes per launch vs the algorithmic bytes of DESIGN.md §6 (within 5%)."""
import csv
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = {"c4": (256 ** 3, 7 * 256 ** 3 - 6 * 256 ** 2, 100), "c3": (1024 ** 2, 5 * 1024 ** 2 - 4 * 1024, 300)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def alg(kernel, cfg, p):
    n, nnz, k = CFG[cfg]
    drain = p == k
    if kernel.startswith("bdot"):
        return 8 * n * p + (8 if drain else 16) * n
    if kernel.startswith("update"):
        return 8 * n * p + (16 if drain else 32) * n
    return nnz * 12 + (n + 1) * 4 + 16 * n


def read(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    m = {}
    for r in rows[1:]:
        m[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", "")) * UNIT.get(r[h.index("Metric Unit")], 1)
    return m


def main(src):
    out = ["| kernel | config | p | DRAM bytes | algorithmic bytes | ratio | time µs | DRAM GB/s |",
           "|---|---|---|---|---|---|---|---|"]
    for f in sorted(glob.glob(os.path.join(src, "tr_*_c*_p*.csv")), key=lambda x: (x.split("_")[-2], x)):
        mm = re.match(r"tr_(.+)_(c\d)_p(\d+)\.csv", os.path.basename(f))
        kernel, cfg, p = mm.group(1), mm.group(2), int(mm.group(3))
        m = read(f)
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        a = alg(kernel, cfg, p)
        t = m["gpu__time_duration.sum"]
        out.append(f"| `{kernel}` | {cfg} | {p} | {dram:.4g} | {a:.4g} | {dram / a:.3f} | {t * 1e6:.1f} | {dram / t / 1e9:.0f} |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"))
