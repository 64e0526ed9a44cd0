#!/usr/bin/env python3
"""One persistent-kernel cycle (c1 or c2, Alg. 3 or IGS(1)) for ncu: python tools/pc_one.py c2 igs2"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, workloads as W, paper_2205_07805_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
alg = sys.argv[2] if len(sys.argv) > 2 else "igs2"
prob = W.config(cfg)
s = P.Solver(prob.A)
b = torch.from_numpy(prob.b).cuda()
for _ in range(2):
    r = s.solve(b, k=prob.k, algorithm=alg, want_H=False)
torch.cuda.synchronize()
print(cfg, alg, r["iters"], r["term"])
s.close()
