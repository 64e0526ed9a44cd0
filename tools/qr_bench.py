#!/usr/bin/env python3
"""Algorithm 1 (igs_qr) throughput on the device: A (n x m) random, two and one sweeps;
algorithmic bytes per column k >= 2: block dot 8 n k (+16 n) and update 8 n k (+32 n), two
sweeps add the same again for the second reduction."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_07805_b200 as P
    for n, m in ((1 << 20, 100), (1 << 22, 50), (16 * 1024 * 1024, 30)):
        ld = n
        A = torch.randn(m * ld, dtype=torch.float64, device="cuda")
        Q = torch.empty_like(A)
        R = torch.empty(m * m, dtype=torch.float64, device="cuda")
        for sweeps in (2, 1):
            P.igs_qr(n, m, A, ld, Q, ld, R, sweeps)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 3
            for _ in range(reps):
                red = P.igs_qr(n, m, A, ld, Q, ld, R, sweeps)
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / reps
            by = sum(16.0 * n * k + 48.0 * n for k in range(1, m)) * (2 if sweeps == 2 else 1)
            G = (Q.view(m, ld)[:, :n]).double()
            loo = torch.linalg.norm(torch.eye(m, device="cuda", dtype=torch.float64) - G @ G.T).item()
            print(json.dumps({"n": n, "m": m, "sweeps": sweeps, "ms": t * 1e3, "reductions": red,
                              "gbs_model": by / t / 1e9, "loo": loo}))


if __name__ == "__main__":
    main()
