#!/usr/bin/env python3
"""c4 GMRES(100) to a true relative residual of 1e-12 (BASELINE config 4 as specified):
wall time of the igs_solve call alone (device-resident b/x, after one warm-up cycle),
iterations, cycles, achieved it/s, and the per-kernel split of a second, timed run.

  python tools/full_solve.py [--config c4] [--alg igs2] [--tol 1e-12]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--alg", default="igs2")
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--kmax", type=int, default=3000)
    a = ap.parse_args()
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config(a.config)
    restart = prob.restart or 100
    s = P.Solver(prob.A)
    b = torch.from_numpy(prob.b).cuda()
    s.solve(b, k=restart, restart=restart, tol=0.0, algorithm=a.alg, want_H=False)   # warm-up cycle
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    r = s.solve(b, k=a.kmax, restart=restart, tol=a.tol, algorithm=a.alg, want_H=False)
    e1.record()
    e1.synchronize()
    wall = time.perf_counter() - t0
    dev = e0.elapsed_time(e1) / 1e3
    s.set_timing(2)
    s.solve(b, k=a.kmax, restart=restart, tol=a.tol, algorithm=a.alg, want_H=False)
    ks = s.kernel_stats()
    s.close()
    out = {"config": a.config, "alg": a.alg, "tol": a.tol, "iters": r["iters"], "cycles": r["cycles"],
           "term": r["term"], "true_relres": r["true_relres"], "wall_s": wall, "device_s": dev,
           "it_s": r["iters"] / dev,
           "kernels_ms": {k: round(v["ms"], 1) for k, v in ks.items() if v["launches"]}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
