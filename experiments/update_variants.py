#!/usr/bin/env python3
"""Run igs_op_update on fixed seeded inputs and print a SHA-256 of the outputs (used by
tests/test_gpu_kernels.py to check the bulk-copy update kernel is bitwise equal to the
register kernel: run once with IGS_UPDATE_TMA=0 and once with =1)."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_07805_b200 as P
    h = hashlib.sha256()
    for n, p, gs in [(512, 8, 2), (70001, 9, 1), (70001, 37, 2), (1 << 20, 64, 2), (1 << 20, 100, 1), (5003, 300, 2)]:
        rng = np.random.default_rng(n + p + gs)
        ld = n + (n % 2) + 32
        Vh = np.zeros((p + 2, ld)); Vh[:, :n] = rng.standard_normal((p + 2, n))
        z = np.zeros(ld); z[:n] = rng.standard_normal(n)
        alpha = rng.standard_normal(p) * 1e-3 if gs == 2 else None
        beta = rng.standard_normal(p + 1)
        Vd = torch.from_numpy(Vh.reshape(-1)).cuda()
        zd = torch.from_numpy(z).cuda()
        ad = torch.from_numpy(alpha).cuda() if alpha is not None else None
        bd = torch.from_numpy(beta).cuda()
        for want_next in (True, False):
            W = Vd.clone()
            P.igs_op_update(n, p, W, ld, W[p * ld:], zd, ad, bd, 0.75, W[p * ld:],
                            W[(p + 1) * ld:] if want_next else None)
            h.update(W.cpu().numpy().tobytes())
    print(h.hexdigest())


if __name__ == "__main__":
    main()
