#!/usr/bin/env python3
"""Dump H and x of a few solves (npz) for bitwise A/B comparison of compile variants:
python tools/tri_ab.py out.npz"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2205_07805_b200 as P, workloads as W
res = {}
for cfg, alg, persist in (("c1", "igs1", "1"), ("c2", "igs1", "1"), ("c2", "igs2", "1"), ("c1", "igs2_two", "0"),
                          ("c2", "igs1", "0"), ("c2", "igs2", "0")):
    os.environ["IGS_PERSIST"] = persist
    prob = W.config(cfg)
    s = P.Solver(prob.A)
    g = s.solve(torch.from_numpy(prob.b).cuda(), k=prob.k, algorithm=alg)
    s.close()
    key = f"{cfg}_{alg}_{persist}"
    res[key + "_H"] = g["H"]
    res[key + "_x"] = g["x"].cpu().numpy()
np.savez(sys.argv[1], **res)
print("saved", len(res))
