#!/usr/bin/env python3
"""Persistent cycle kernel vs the graph-replayed per-kernel path across problem sizes: the
evidence for the default thresholds (igs_ctx::pc_max_n per algorithm and cycle length).

For each c3-shaped 2D stencil (N^2 rows) and each (algorithm, cycle length m) it times one
unrestarted cycle of m iterations both ways (IGS_PERSIST=1 with the threshold lifted, and
IGS_PERSIST=0) in a fresh process, best of --reps, and prints one JSON line per size.

  python tools/pc_crossover.py [--Ns 300,362,384,400,420,434,443,460,470,512] [--algs igs1,igs2]
                              [--ms 100,300] [--reps 3]
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
N, alg, m, reps = %d, %r, %d, %d
prob = W.config("c3", N=N)
s = P.Solver(prob.A)
b = torch.from_numpy(prob.b).cuda()
s.solve(b, k=m, algorithm=alg, want_H=False)
best = None
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = s.solve(b, k=m, algorithm=alg, want_H=False); e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1)
    best = t if best is None else min(best, t)
info = s.info()
print(json.dumps({"it_s": r["iters"] / (best / 1e3), "pcycle": info["pcycle_launches"] > 0}))
"""


def run(N, alg, m, reps, persist):
    env = dict(os.environ, IGS_PERSIST=str(persist), IGS_PC_MAX_N="100000000")
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, N, alg, m, reps)], env=env, capture_output=True,
                       text=True, timeout=600)
    if r.returncode != 0:
        return {"error": r.stderr[-400:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Ns", default="300,362,384,400,420,434,443,460,470,512")
    ap.add_argument("--algs", default="igs1,igs2")
    ap.add_argument("--ms", default="100,300")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for m in [int(x) for x in a.ms.split(",")]:
        for alg in a.algs.split(","):
            for N in [int(x) for x in a.Ns.split(",")]:
                pc, gr = run(N, alg, m, a.reps, 1), run(N, alg, m, a.reps, 0)
                print(json.dumps({"N": N, "n": N * N, "alg": alg, "m": m, "persistent": pc, "graphs": gr,
                                  "ratio": (pc.get("it_s", 0) / gr["it_s"]) if gr.get("it_s") else None}),
                      flush=True)


if __name__ == "__main__":
    main()
