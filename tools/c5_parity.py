#!/usr/bin/env python3
"""Config c5 (512^3 stencil, int64 columns, n = 134M) on one GPU against the oracle on the
same inputs, k = 30 (the host holds the oracle's basis only for a short
cycle): Hessenberg column-normwise difference over the 30 columns and the Arnoldi residual
history.  A one-off record for BASELINE.md (slow on the host), not a test."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import oracle
    import paper_2205_07805_b200 as P
    import workloads as W
    k = 30
    prob = W.config("c5")
    s = P.Solver(prob.A)
    t0 = time.time()
    g = s.solve(torch.from_numpy(prob.b).cuda(), k=k, gs_iters=2)
    tg = time.time() - t0
    s.close()
    del s
    torch.cuda.empty_cache()
    t0 = time.time()
    o = oracle.gmres(prob.A, prob.b, k, variant="igs2", dot_block=4096)
    to = time.time() - t0
    d = oracle.column_normwise_diff(g["H"], o["H"], k)
    rg, ro = np.asarray(g["res_hist"]), np.asarray(o["res_hist"])
    print(json.dumps({"config": "c5", "k": k, "n": prob.A.n_rows, "nnz": prob.A.nnz,
                      "gpu_iters": g["iters"], "oracle_iters": o["iters"], "H_colnormwise": d,
                      "res_hist_max_rel": float(np.max(np.abs(rg - ro) / ro)),
                      "gpu_wall_s": tg, "oracle_wall_s": to}))


if __name__ == "__main__":
    main()
