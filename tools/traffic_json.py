#!/usr/bin/env python3
"""ncu per-launch DRAM bytes (tools/profile_traffic.sh) -> profiles/ncu_traffic.json with the
ratio DRAM bytes / algorithmic bytes of the same launch (c4, p = 50; DESIGN.md byte model)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 256 ** 3
NNZ = 7 * 256 ** 3 - 6 * 256 ** 2
P = 50
ALG = {  # algorithmic bytes of the launch at iteration p
    "block_dot": 8 * N * P + 16 * N,
    "update": 8 * N * P + 32 * N,
    "spmv": NNZ * 12 + (N + 1) * 4 + 16 * N,
}
FILES = {"block_dot": "traffic_bdot.csv", "update": "traffic_update.csv", "spmv": "traffic_spmv.csv"}
# round 2 (tools/r2_call23.sh): python tools/traffic_json.py profiles/r2/c23/traffic c23_tr_
R2 = {"block_dot": "bdot_tma_kernel_c4_p50.csv", "update": "update_kernel_c4_p50.csv",
      "spmv": "spmv_sell_diag_kernel_c4_p50.csv"}
# bytes one c4 SpMV streams in the stored format (SELL-32, every slice diagonal, stored by list
# position; igs_info "spmv_bytes", profiles/r2/c23/c23_c4_info.json)
SPMV_STORED = 1260388360
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def read(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    out = {}
    for r in rows[1:]:
        out[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", "")) * UNIT.get(r[h.index("Metric Unit")], 1)
    return out, r[h.index("Kernel Name")].split("(")[0]


def main(src, prefix=None):
    res = {"_about": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none on one launch at iteration p = 50 of a c4 Alg. 3 solve "
                     f"({'tools/r2_call23.sh, ' + os.path.relpath(src, ROOT) if prefix else 'tools/profile_traffic.sh'}); "
                     "ratio = DRAM bytes / algorithmic bytes (the SpMV's algorithmic bytes are the CSR "
                     "definition of SURVEY 8(d); stored_bytes = what the SELL copy streams)"}
    for k, f in (R2 if prefix else FILES).items():
        m, name = read(os.path.join(src, (prefix or "") + f))
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        res[k] = {"kernel": name, "p": P, "dram_bytes": dram, "alg_bytes": ALG[k], "ratio": dram / ALG[k],
                  "time_s": m["gpu__time_duration.sum"], "dram_gbs": dram / m["gpu__time_duration.sum"] / 1e9}
        if k == "spmv" and prefix:
            res[k]["stored_bytes"] = SPMV_STORED
            res[k]["ratio_stored"] = dram / SPMV_STORED
    json.dump(res, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"),
         sys.argv[2] if len(sys.argv) > 2 else None)
