#!/usr/bin/env python3
"""Summarise ncu outputs for profiles/: a launch-list CSV (gpu__time_duration.sum per
launch) -> per-kernel share table; a --set full report -> per-launch DRAM bytes, time,
achieved DRAM GB/s, occupancy and top stall reasons."""
import collections
import csv
import io
import subprocess
import sys


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {t:.0f} | {100 * t / tot:.1f}% |")
    return "\n".join(out)


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(h)}

    def g(r, n):
        i = col.get(n)
        return r[i] if i is not None else ""

    def num(r, n):
        try:
            return float(g(r, n).replace(",", ""))
        except ValueError:
            return float("nan")

    def tobytes(r, n):
        u = units[col[n]] if n in col else ""
        v = num(r, n)
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    def tosec(r, n):
        u = units[col[n]] if n in col else ""
        return num(r, n) * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1)

    out = ["| kernel | grid | time us | DRAM read GB | DRAM write GB | DRAM GB/s | DRAM % peak | regs | warps active % |",
           "|---|---|---|---|---|---|---|---|---|"]
    for r in data:
        name = g(r, "Kernel Name").split("(")[0].replace("void ", "")
        t = tosec(r, "gpu__time_duration.sum")
        rd, wr = tobytes(r, "dram__bytes_read.sum"), tobytes(r, "dram__bytes_write.sum")
        out.append(f"| `{name}` | {g(r, 'Grid Size')} | {t * 1e6:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                   f"{(rd + wr) / t / 1e9:.0f} | {g(r, 'FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed') or g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{g(r, 'launch__registers_per_thread')} | {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')} |")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"\n### {p}\n")
        print(launch_shares(p) if p.endswith(".csv") else full_report(p))
