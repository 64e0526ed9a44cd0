#!/usr/bin/env python3
"""Block-dot bandwidth vs p and leading dimension (isolated launches, CUDA events).

  python tools/bdot_probe.py [--n 1048576] [--ps 10,50,100,200,300] [--pads 0,32] [--reps 10]

Algorithmic bytes per launch: 8 n p (V_p) + 16 n (u, z).  Prints one JSON line per case.
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
            print(json.dumps({"n": n, "ld": ld, "p": p, "us": ms * 1e3, "gbs": by / (ms / 1e3) / 1e9}), flush=True)
        del V


if __name__ == "__main__":
    main()
