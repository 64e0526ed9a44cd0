#!/usr/bin/env python3
"""One c4 solve of k = 60 iterations (no restart) for ncu: the n-th launch of each
iteration kernel is iteration p = n (see tools/profile_traffic.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config("c4")
    s = P.Solver(prob.A)
    r = s.solve(torch.from_numpy(prob.b).cuda(), k=60, gs_iters=2, want_H=False)
    print("iters", r["iters"], "relres", r["true_relres"])
    s.close()


if __name__ == "__main__":
    main()
