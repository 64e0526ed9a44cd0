#!/usr/bin/env python3
"""One-GPU proxy of a c4 rank at G = 8: the 128^3 stencil (n = 2,097,152 = one 32-plane
z-slab of 256^3) through one GMRES(100) cycle, on the plain single-GPU path and on the two
G > 1 reduction paths with a 1-rank communicator (IGS_XCHG=1: the fused exchange in the
block dot; IGS_FORCE_NCCL=1: ncclAllReduce after every block dot), and with the two outer
planes routed through the boundary pass of the split SpMV (IGS_TEST_BND_ENDS: the interior
rows on the main stream, the 2 n / 32 boundary rows by the row-list kernel on the halo stream,
fork / join inside the captured cycle -- everything a rank does at G > 1 but the transports).  Reports it/s, the byte
model's GB/s and the per-iteration time next to the HBM ideal -- the per-iteration overhead
budget of SURVEY §8(e) (80% strong scaling at 8 GPUs needs <= 60-72 us of it).

  python tools/slab_proxy.py [--N 128] [--reps 5] [--gs 2]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import torch
import paper_2205_07805_b200 as P
import workloads as W
N, reps, gs = %d, %d, %d
prob = W.config("c4", N=N)
s = P.Solver(prob.A)
b = torch.from_numpy(prob.b).cuda()
for _ in range(2):
    s.solve(b, k=100, restart=100, gs_iters=gs, want_H=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
it = 0
for _ in range(reps):
    it += s.solve(b, k=100, restart=100, gs_iters=gs, want_H=False)["iters"]
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"it_s": it / (ms / 1e3), "ms_per_cycle": ms / reps, "info": s.info()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gs", type=int, default=2)
    a = ap.parse_args()
    n = a.N ** 3
    nnz = 7 * n - 6 * a.N * a.N
    model = sum(nnz * 12 + (n + 1) * 4 + 16 * n + 16 * n * p for p in range(1, 101))
    out = {"N": a.N, "n": n}
    plane = str(n // 32)  # a c4 z-slab at G = 8 is 32 planes thick: each outer plane holds n / 32 rows
    for name, env in (("plain", {}), ("xchg_1rank", {"IGS_XCHG": "1"}), ("ncclallreduce_1rank", {"IGS_FORCE_NCCL": "1"}),
                      ("split_spmv", {"IGS_TEST_BND_ENDS": plane}),
                      ("split_spmv_xchg_1rank", {"IGS_TEST_BND_ENDS": plane, "IGS_XCHG": "1"})):
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.N, a.reps, a.gs)], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            out[name] = {"error": r.stderr[-500:]}
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        d["gbs_model"] = model / (d["ms_per_cycle"] / 1e3) / 1e9
        d["us_per_iteration"] = d["ms_per_cycle"] * 10.0
        d["hbm_ideal_us_per_iteration_at_6555"] = model / 100 / 6554.9e9 * 1e6
        out[name] = d
    print(json.dumps(out))


if __name__ == "__main__":
    main()
