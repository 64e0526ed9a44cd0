#!/usr/bin/env python3
"""igs_op_trisolve latency for orders 1..300 (call + launch + sync), for the small-step
forward-substitution experiments."""
import os
import sys

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
for order in (1, 32, 64, 128, 256, 300):
    for _ in range(3): P.igs_op_trisolve(order, Ld, M, b, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(50): P.igs_op_trisolve(order, Ld, M, b, x)
    e1.record(); e1.synchronize()
    print(order, round(e0.elapsed_time(e1) / 50 * 1000, 1), 'us per call (incl. launch + sync)')
