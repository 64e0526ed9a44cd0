#!/usr/bin/env python3
"""One unrestarted Alg. 3 solve for ncu (default c4, k = 60): the n-th launch of each
iteration kernel is iteration p = n (see tools/profile_traffic_v3.sh for the skip counts).

  python tools/traffic_run.py [--config c4] [--k 60] [--alg igs2_two]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--k", type=int, default=60)
    ap.add_argument("--alg", default=None, help="igs1 | igs2 | igs2_two | mgs (default: Alg. 3)")
    a = ap.parse_args()
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config(a.config)
    s = P.Solver(prob.A)
    r = s.solve(torch.from_numpy(prob.b).cuda(), k=a.k, gs_iters=2, want_H=False, algorithm=a.alg)
    print("iters", r["iters"], "relres", r["true_relres"])
    s.close()


if __name__ == "__main__":
    main()
