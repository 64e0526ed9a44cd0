#!/usr/bin/env python3
"""Second solve-gap probe: the c4 solve as specified (tol 1e-12) twice, against the same
iteration count without a tolerance, and the cycle count / iterations of each."""
import json
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
    b = torch.from_numpy(prob.b).cuda()
    s.solve(b, k=100, restart=100, tol=0.0, want_H=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k, tol in ((3000, 1e-12), (3000, 1e-12), (1246, 0.0), (1200, 1e-12), (1300, 1e-11)):
        e0.record()
        r = s.solve(b, k=k, restart=100, tol=tol, want_H=False)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"k": k, "tol": tol, "iters": r["iters"], "cycles": r["cycles"], "term": r["term"],
                          "ms": ms, "it_s": r["iters"] / (ms / 1e3)}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
