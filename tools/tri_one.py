#!/usr/bin/env python3
"""One igs_op_trisolve of order 300 after a warm-up (for ncu -k regex:trisolve)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2205_07805_b200 as P
rng = np.random.default_rng(0)
M = 320
L = np.tril(rng.uniform(-1, 1, (M, M)), -1) * 1e-2
Ld = torch.from_numpy(np.asfortranarray(L).reshape(-1, order="F")).cuda()
b = torch.from_numpy(rng.standard_normal(M)).cuda()
x = torch.empty(M, dtype=torch.float64, device='cuda')
for _ in range(3):
    P.igs_op_trisolve(300, Ld, M, b, x)
torch.cuda.synchronize()
print("ok")
