#!/usr/bin/env python3
"""Time igs_solve on any BASELINE config (c1..c5) on one GPU: Arnoldi it/s, achieved GB/s
under the SURVEY §8(d) byte model, per-kernel split.  Not the driver's bench (bench.py is);
this fills BASELINE.md's per-config table.

  python tools/bench_configs.py --config c3 [--gs 2] [--k 300] [--reps 3]
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
    ap.add_argument("--config", default="c3")
    ap.add_argument("--gs", type=int, default=2)
    ap.add_argument("--alg", default=None, help="igs1 | igs2 | igs2_two | mgs (overrides --gs)")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--restart", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--N", type=int, default=0)
    args = ap.parse_args()
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config(args.config, N=args.N or None)
    k = args.k or (prob.k if prob.restart == 0 else prob.restart)
    restart = prob.restart if args.restart < 0 else args.restart
    if restart and restart < k:
        k = restart
    A = prob.A
    n, nnz = A.n_rows, A.nnz
    sc = 8 if A.colind.dtype.itemsize == 8 else 4
    s = P.Solver(A)
    b = torch.from_numpy(prob.b).cuda()
    s.solve(b, k=k, restart=0, tol=0.0, gs_iters=args.gs, want_H=False, algorithm=args.alg)
    torch.cuda.synchronize()
    def timed(timing):
        s.set_timing(2 if timing else 0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it = 0
        for _ in range(args.reps):
            r = s.solve(b, k=k, restart=0, tol=0.0, gs_iters=args.gs, want_H=False, algorithm=args.alg)
            it += r["iters"]
        e1.record()
        e1.synchronize()
        return it, e0.elapsed_time(e1), r
    it, ms, r = timed(False)          # the number (CUDA graphs allowed)
    _, ms_t, _ = timed(True)          # per-kernel split (events around every launch)
    ks = s.kernel_stats()
    s.set_timing(0)
    b_spmv = nnz * (8 + sc) + (n + 1) * (8 if sc == 8 else 4) + 16 * n
    model = args.reps * sum(b_spmv + 16 * n * p for p in range(1, k + 1))
    out = {"config": args.config, "gs": args.gs, "alg": args.alg or {1: "igs1", 2: "igs2"}[args.gs],
           "reductions_per_solve": r["reductions"], "n": n, "nnz": nnz, "k": k, "reps": args.reps,
           "it_s": it / (ms / 1e3), "ms_per_solve": ms / args.reps,
           "gbs_model": model / (ms / 1e3) / 1e9, "ms_per_solve_timed_run": ms_t / args.reps,
           "kernels": {kk: {"ms": v["ms"] / args.reps, "launches": v["launches"] / args.reps,
                            "gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 and v["bytes"] else None}
                       for kk, v in ks.items() if v["launches"]}}
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
