#!/usr/bin/env python3
"""Oracle-only reference records for the full-size parity tests (tests/golden/oracle_*.json).

Calls only oracle/ and workloads/ (the seeded input generators): nothing here touches the
CUDA path, so the stored values are the oracle's.  Slow -- run once, commit
the JSON:

  python tools/oracle_records.py c4 --gs 2     # BASELINE configs[3] as specified:
                                               # GMRES(100) to 1e-12 (~20 min on 16 cores)
  python tools/oracle_records.py c5            # configs[4]: k = 100 unrestarted, V = 108 GB
                                               # (needs ~130 GB of host RAM)

Each record: iterations, cycles, termination, true relative residual, the Givens-recurrence
residual history, ||A||_2 (power iteration on A^T A, S:76-84 / reading R11), the backward
error beta(x) = ||b - A x|| / (||b|| + ||A||_2 ||x||), and for c5 the first 30
Hessenberg columns and ||I - V^T V||_F.
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
    ap.add_argument("config", choices=["c4", "c5"])
    ap.add_argument("--gs", type=int, default=2, choices=[1, 2])
    ap.add_argument("--norm-maxit", type=int, default=500)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import oracle
    import workloads as W
    oracle.build()
    var = {1: "igs1", 2: "igs2"}[a.gs]
    t0 = time.time()
    prob = W.config(a.config)
    t_gen = time.time() - t0
    rec = {"config": a.config, "gs": a.gs, "variant": var, "n": prob.A.n_rows, "nnz": prob.A.nnz,
           "oracle_threads": oracle.num_threads(), "written_by": "tools/oracle_records.py (oracle/ only)"}
    # memory order for c5 (V = 108 GB on a 196 GB host): the solve and the LOO first (the Gram
    # in row blocks, no second copy of V), then V is dropped before ||A||_2 (scipy copy of A)
    t0 = time.time()
    if a.config == "c4":
        o = oracle.gmres(prob.A, prob.b, 3000, restart=100, tol=1e-12, variant=var, dot_block=4096)
        rec.update(k=3000, restart=100, tol=1e-12, dot_block=4096)
    else:
        # block sums added pairwise (reading R27): at 134M rows a running sum over 32K block
        # sums puts ~3.6e-12 of rounding into every inner product and into the basis' LOO
        o = oracle.gmres(prob.A, prob.b, 100, restart=0, tol=0.0, variant=var, dot_block=-4096, want_V=True)
        rec.update(k=100, restart=0, tol=0.0, dot_block=-4096)
    t_solve = time.time() - t0
    rec.update(iters=o["iters"], cycles=o["cycles"], term=o["term"], true_relres=o["true_relres"],
               basis_cols=o["basis_cols"], res_hist=[float(v) for v in o["res_hist"]],
               x_norm=float(np.linalg.norm(o["x"])))
    if a.config == "c5":
        c = o["basis_cols"]
        t1 = time.time()
        rec["loo"] = oracle.loss_of_orthogonality(o["V"][:, :c], row_block=4096)
        rec["t_loo_s"] = time.time() - t1
        rec["H_first30"] = o["H"][:31, :30].T.tolist()  # column j = H[:31, j]
        del o["V"]
    t0 = time.time()
    normA = oracle.norm2_estimate(prob.A, maxit=a.norm_maxit)
    t_norm = time.time() - t0
    rec.update(normA_2=normA, normA_maxit=a.norm_maxit, beta=oracle.backward_error(prob.A, prob.b, o["x"], normA))
    import resource
    rec.update(t_generate_s=t_gen, t_norm_s=t_norm, t_solve_s=t_solve,
               host_peak_rss_gb=resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6)
    out = a.out or os.path.join(ROOT, "tests", "golden", f"oracle_{a.config}_gs{a.gs}.json")
    with open(out, "w") as f:
        json.dump(rec, f)
    print(json.dumps({k: v for k, v in rec.items() if k not in ("res_hist", "H_first30")}))


if __name__ == "__main__":
    main()
