#!/usr/bin/env python3
"""Where the full c4 solve loses time against the one-cycle bench step: device time of
igs_solve for c GMRES(100) cycles (tol = 0, exactly c*100 iterations) and with a tolerance
that is never reached (tol = 1e-30), next to the per-cycle time of the one-cycle step.

  python tools/solve_gap.py [--config c4] [--cycles 1,2,4,8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--cycles", default="1,2,4,8")
    a = ap.parse_args()
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    prob = W.config(a.config)
    s = P.Solver(prob.A)
    b = torch.from_numpy(prob.b).cuda()
    s.solve(b, k=100, restart=100, tol=0.0, want_H=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for c in [int(x) for x in a.cycles.split(",")]:
        for tol in (0.0, 1e-30):
            e0.record()
            r = s.solve(b, k=100 * c, restart=100, tol=tol, want_H=False)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            print(json.dumps({"cycles": c, "tol": tol, "iters": r["iters"], "ms": ms, "ms_per_cycle": ms / c,
                              "it_s": r["iters"] / (ms / 1e3)}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
