import os, sys
sys.path.insert(0, "/root/repo")
import torch, workloads as W, paper_2205_07805_b200 as P
prob = W.config("c3", N=64)
b = torch.from_numpy(prob.b).cuda()
for env in ({"IGS_PC_NTRI": "2"}, {"IGS_PC_NTRI": "1"}, {"IGS_PERSIST": "0"}):
    for kk in ("IGS_PC_NTRI", "IGS_PERSIST"): os.environ.pop(kk, None)
    os.environ.update(env); os.environ["IGS_PC_MAX_N"] = "100000"
    for grid in ("0", "4"):
        os.environ["IGS_PC_GRID"] = grid
        s = P.Solver(prob.A)
        for (k, r, t) in ((400, 150, 1e-8), (70, 30, 1e-10), (200, 0, 1e-9)):
            g = s.solve(b, k=k, restart=r, tol=t, gs_iters=2)
            print(env, grid, (k, r, t), g["iters"], g["term"], g["cycles"], g["reductions"])
        s.close()
