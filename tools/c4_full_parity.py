#!/usr/bin/env python3
"""Config c4 exactly as specified (256^3, GMRES(100) to a true relative residual of 1e-12) on
the GPU and in the oracle on the same inputs: iterations, cycles, final true residual, and
the Arnoldi residual at every cycle start.  Slow (the oracle streams ~15 GB per iteration on
the host); a one-off record for BASELINE.md, not a test.

  python tools/c4_full_parity.py [--gs 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gs", type=int, default=2)
    a = ap.parse_args()
    import torch
    import oracle
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config("c4")
    var = {1: "igs1", 2: "igs2"}[a.gs]
    s = P.Solver(prob.A)
    t0 = time.time()
    g = s.solve(torch.from_numpy(prob.b).cuda(), k=3000, restart=100, tol=1e-12, gs_iters=a.gs, want_H=False)
    tg = time.time() - t0
    s.close()
    t0 = time.time()
    o = oracle.gmres(prob.A, prob.b, 3000, restart=100, tol=1e-12, variant=var, dot_block=4096)
    to = time.time() - t0
    rg, ro = np.asarray(g["res_hist"]), np.asarray(o["res_hist"])
    m = min(len(rg), len(ro))
    starts = list(range(0, m, 100))
    out = {"gs": a.gs, "gpu": {"iters": g["iters"], "cycles": g["cycles"], "term": g["term"],
                               "true_relres": g["true_relres"], "wall_s": tg},
           "oracle": {"iters": o["iters"], "cycles": o["cycles"], "term": o["term"],
                      "true_relres": o["true_relres"], "wall_s": to},
           "res_hist_at_cycle_starts": [[int(i), float(rg[i]), float(ro[i])] for i in starts],
           "max_rel_diff_res_hist": float(np.max(np.abs(rg[:m] - ro[:m]) / np.maximum(ro[:m], 1e-300)))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
