#!/usr/bin/env python3
"""Small invocations of every device path (an all-path smoke; meant for compute-sanitizer,
which this GPU pool does not allow): persistent cycle kernel, graph-replayed cycles, the per-kernel path (both gs,
two-reduce, MGS), the bulk-copy block dot at a few sizes, SELL and CSR SpMV, QR,
basis diagnostics.  Exit code 0 = every call returned IGS_OK."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_07805_b200 as P
    import workloads as W
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    prob = W.config("c1")
    s = P.Solver(prob.A)
    b = torch.from_numpy(prob.b).cuda()
    for gs in (1, 2):
        s.solve(b, k=40, gs_iters=gs, want_loo=True, want_diag=True)          # persistent kernel
    s.close()
    os.environ["IGS_PERSIST"] = "0"
    prob = W.config("c3", N=40)                                                 # n = 1600
    s = P.Solver(prob.A)
    b = torch.from_numpy(prob.b).cuda()
    for alg in ("igs2", "igs1", "igs2_two", "mgs"):
        s.solve(b, k=30, restart=12, tol=1e-10, algorithm=alg, want_loo=True)   # graphs
    s.set_timing(1)
    for alg in ("igs2", "igs1"):
        s.solve(b, k=30, restart=12, tol=1e-10, algorithm=alg)                  # stream path
    s.set_timing(0)
    s.close()
    if which == "all":
        rng = np.random.default_rng(0)
        for n, p in ((700, 9), (1537, 17), (5000, 40)):
            ld = n + (n % 2)
            V = torch.from_numpy(rng.standard_normal((p + 2) * ld)).cuda()
            z = torch.from_numpy(rng.standard_normal(ld)).cuda()
            out = torch.empty(2 * (p + 1), dtype=torch.float64, device="cuda")
            P.igs_op_block_dot(n, p, V, ld, V[p * ld:], z, out)
            P.igs_op_basis_diag(n, p, V, ld)
            A = torch.from_numpy(rng.standard_normal(ld * p)).cuda()
            Q = torch.empty(ld * p, dtype=torch.float64, device="cuda")
            R = torch.empty(p * p, dtype=torch.float64, device="cuda")
            P.igs_qr(n, p, A, ld, Q, ld, R, 2)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
