#!/usr/bin/env python3
"""Block-dot and fused-update bandwidth vs p and leading dimension (isolated back-to-back
launches, CUDA events; igs_bench_block_dot / igs_bench_update).

  python tools/bdot_probe.py [--n 1048576] [--ps 10,50,100,200,300] [--pads 0,32] [--reps 10]

Algorithmic bytes per launch: block dot 8 n p + 16 n (V_p, u, z); Alg. 3
update 8 n p + 32 n (V_p, u, z read; v_p, u' written).  One JSON line per case.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--ps", default="10,50,100,200,300")
    ap.add_argument("--pads", default="0,32")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import paper_2205_07805_b200 as P
    n = a.n
    ps = [int(x) for x in a.ps.split(",")]
    pmax = max(ps)
    for pad in [int(x) for x in a.pads.split(",")]:
        ld = n + pad
        V = torch.rand(ld * pmax, dtype=torch.float64, device="cuda")
        u = torch.rand(n, dtype=torch.float64, device="cuda")
        z = torch.rand(n, dtype=torch.float64, device="cuda")
        out = torch.empty(2 * (pmax + 1), dtype=torch.float64, device="cuda")
        for p in ps:
            ms = P.igs.igs_bench_block_dot(n, p, V, ld, u, z, out, reps=a.reps)
            by = 8.0 * n * p + 16.0 * n
            coef = torch.rand(p + 1, dtype=torch.float64, device="cuda") * 1e-3
            vo = torch.empty(n, dtype=torch.float64, device="cuda")
            un = torch.empty(n, dtype=torch.float64, device="cuda")
            ms_u = P.igs.igs_bench_update(n, p, V, ld, u, z, coef, coef, 1.5, vo, un, reps=a.reps)
            by_u = 8.0 * n * p + 32.0 * n
            print(json.dumps({"n": n, "ld": ld, "p": p, "bdot_us": ms * 1e3, "bdot_gbs": by / (ms / 1e3) / 1e9,
                              "update_us": ms_u * 1e3, "update_gbs": by_u / (ms_u / 1e3) / 1e9}), flush=True)
        del V


if __name__ == "__main__":
    main()
