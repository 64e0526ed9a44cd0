#!/usr/bin/env python3
"""bench.py -- Arnoldi iterations/s and achieved HBM GB/s of the IGS-GMRES hot path on B200.

Workload (BASELINE.json configs[3], "c4"): 3D convection-diffusion 7-point stencil on a
256^3 grid (n = 16,777,216, nnz = 117,047,296, CSR FP64, int32 columns), convection
(100,50,25), b ~ U(0,1) seed 3, x0 = 0, GMRES(100).  One "step" = one restart cycle of 100
Arnoldi iterations through igs_solve (k = restart = 100, tol = 0, gs_iters = 2 = Alg. 3):
||b||, r0, priming, 100 x [SpMV, fused block dot, (allreduce), small step, fused update],
least squares, x += V y, final residual.  value = Arnoldi iterations (all ranks' one shared
Krylov process) per second; the basis V (13.6 GB) is far larger than L2, so no flush is
needed between steps.  N > 1: the same 256^3 problem row-block sharded over N ranks
(strong scaling), one NCCL allreduce of 2(p+1) doubles per iteration + halo send/recv.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, plain FP64 C + OpenMP) on the host cores,
rank 0 only; each step is a bounded sample (the first 50 Arnoldi iterations of the same
cycle), projected to the cycle-average iteration with the byte model of DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Arnoldi iterations/s and achieved HBM GB/s (fraction of roofline) at 1/2/4/8 B200"
UNIT = "Arnoldi iterations/s"
N_GRID = 256
M = 100                     # GMRES(100)
CPU_SAMPLE_ITERS = 50       # oracle sample: iterations 1..50 of the cycle (~10 s on 16 cores)


def bench_config(gs: int, world: int) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": f"c4: 3D 7-point convection-diffusion 256^3, GMRES(100) cycle, gs_iters={gs} "
                        f"({'Alg. 3' if gs == 2 else 'Alg. 2, one sweep'})",
            "n": N_GRID ** 3, "nnz": 7 * N_GRID ** 3 - 6 * N_GRID ** 2, "restart": M,
            "parallelism": f"row-block x{world}", "l2": "inputs larger than L2 (V = 13.6 GB), no flush"}


def byte_model(n: int, nnz: int, p: int, s_col: int = 4, s_ptr: int = 4) -> float:
    """Algorithmic bytes of one Arnoldi iteration:
    one SpMV (values + columns + rowptr + x + y) plus two reads of V_p."""
    b_spmv = nnz * (8 + s_col) + (n + 1) * s_ptr + 8 * n + 8 * n
    return float(b_spmv + 2 * 8 * n * p)


def cycle_avg_bytes(n, nnz, m=M):
    return sum(byte_model(n, nnz, p) for p in range(1, m + 1)) / m


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, 1 GiB copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s; MEASURED_PEAKS.json absent)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0])); smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard_bounds(n, world, rank):
    # contiguous row blocks aligned to whole z-planes
    planes = N_GRID
    p0 = planes * rank // world
    p1 = planes * (rank + 1) // world
    plane = N_GRID * N_GRID
    return p0 * plane, p1 * plane


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle, rank 0 only (the other ranks exit 0)."""
    if rank != 0:
        return 0
    import oracle
    import workloads as W
    prob = W.config("c4")
    A, b = prob.A, prob.b
    n, nnz = A.n_rows, A.nnz
    oracle.build()
    cores = oracle.num_threads()
    sample_bytes = sum(byte_model(n, nnz, p) for p in range(1, CPU_SAMPLE_ITERS + 1))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        o = oracle.gmres(A, b, CPU_SAMPLE_ITERS, restart=M, tol=0.0, variant="igs2" if args.gs == 2 else "igs1",
                         dot_block=4096)
        dt = time.perf_counter() - t0
        assert o["iters"] == CPU_SAMPLE_ITERS
        if i >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    gbs = sample_bytes / t / 1e9
    val = gbs * 1e9 / cycle_avg_bytes(n, nnz)            # projected to the cycle average
    sample = (f"oracle gs_iters={args.gs}, first {CPU_SAMPLE_ITERS} Arnoldi iterations of the c4 "
              f"GMRES(100) cycle per step ({t:.1f} s); it/s projected to the 100-iteration cycle "
              f"average by the byte model (sample ran {CPU_SAMPLE_ITERS / t:.3f} it/s, {gbs:.1f} GB/s)")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, workloads/)",
            "config": bench_config(args.gs, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "gbs": gbs, **host_cpu()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def host_cpu() -> dict:
    """Model name and socket count of the host the oracle runs on (/proc/cpuinfo)."""
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and model is None:
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("physical id"):
                    sockets.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"cpu_model": model, "sockets": len(sockets) or None, "nproc": os.cpu_count()}


def cpu_baseline_ours(prob, seconds_cap=40.0):
    """Oracle timed on the host cores beside the GPU run (rank 0, N=1 only)."""
    import oracle
    oracle.build()
    A, b = prob.A, prob.b
    n, nnz = A.n_rows, A.nnz
    t0 = time.perf_counter()
    o = oracle.gmres(A, b, CPU_SAMPLE_ITERS, restart=M, tol=0.0, variant="igs2", dot_block=4096)
    t = time.perf_counter() - t0
    assert o["iters"] == CPU_SAMPLE_ITERS
    sample_bytes = sum(byte_model(n, nnz, p) for p in range(1, CPU_SAMPLE_ITERS + 1))
    gbs = sample_bytes / t / 1e9
    return {"value": gbs * 1e9 / cycle_avg_bytes(n, nnz), "unit": UNIT,
            "cores": oracle.num_threads(), "kind": "oracle",
            "sample": (f"first {CPU_SAMPLE_ITERS} iterations of one c4 GMRES(100) cycle (Alg. 3, "
                       f"blocked FP64 dots), {t:.1f} s wall; projected to the cycle-average "
                       f"iteration by the byte model ({CPU_SAMPLE_ITERS / t:.3f} it/s raw, {gbs:.1f} GB/s)"),
            "gbs": gbs, **host_cpu()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gs", type=int, default=2, choices=[1, 2])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--solve", action="store_true", help="also run one full solve to 1e-12")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2205_07805_b200 as P
    import workloads as W

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_global = N_GRID ** 3
    r0, r1 = shard_bounds(n_global, world, rank) if world > 1 else (0, n_global)
    prob = W.config("c4", row_begin=r0, row_end=r1)
    uid = None
    if world > 1:
        obj = [P.igs_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.current_stream()
    solver = P.Solver(prob.A, device=local, stream=stream, rank=rank, nranks=world, nccl_unique_id=uid)
    n_loc = prob.A.n_rows
    b_dev = torch.from_numpy(prob.b).cuda()
    x_dev = torch.empty(n_loc, dtype=torch.float64, device="cuda")

    def step_dev():
        return solver.solve(b_dev, k=M, restart=M, tol=0.0, gs_iters=args.gs, x_out=x_dev, want_H=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        r = step_dev()
        assert r["iters"] == M, r
    # ---------------- timed region (device, CUDA events on the solver stream) ------------
    clocks = ClockSampler(local)
    solver.set_timing(2)
    barrier()
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0, e1 = ev[0], ev[-1]
    e0.record(stream)
    iters = 0
    for i in range(args.steps):
        iters += step_dev()["iters"]
        ev[i + 1].record(stream)
    e1.synchronize()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    step_ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    ms_median = max_over_ranks(step_ms[len(step_ms) // 2])
    ks = solver.kernel_stats()
    solver.set_timing(0)
    value = iters / (ms / 1e3)
    nnz_g = 7 * N_GRID ** 3 - 6 * N_GRID ** 2
    model_bytes = args.steps * sum(byte_model(n_global, nnz_g, p) for p in range(1, M + 1))
    gbs_iter = model_bytes / (ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    # dominant kernel (largest device time) and its achieved algorithmic GB/s
    dom = max((k for k in ks if ks[k]["launches"] > 0), key=lambda k: ks[k]["ms"])
    dk = ks[dom]
    achieved = dk["bytes"] / (dk["ms"] / 1e3) / 1e9 if dk["ms"] > 0 else 0.0
    launches_per_step = sum(v["launches"] for v in ks.values() if v["launches"]) / args.steps
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            ent = tj.get(dom)
            if ent and ent.get("ratio"):
                traffic = ent["ratio"] * dk["bytes"] / max(dk["launches"], 1)
        except Exception:
            traffic = None
    # ---------------- end-to-end: host buffers, H2D/D2H inside the timed region --------
    e2e = None
    if not args.no_e2e:
        b_host = torch.from_numpy(prob.b).pin_memory()
        x_host = torch.empty(n_loc, dtype=torch.float64).pin_memory()
        solver.solve(b_host, k=M, restart=M, tol=0.0, gs_iters=args.gs, x_out=x_host, want_H=False)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        it2 = 0
        for _ in range(args.steps):
            it2 += solver.solve(b_host, k=M, restart=M, tol=0.0, gs_iters=args.gs, x_out=x_host,
                                want_H=False)["iters"]
        f1.record(stream)
        f1.synchronize()
        barrier()
        ms2 = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": it2 / (ms2 / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n_loc,
               "d2h_bytes_per_step": 8 * n_loc + 8 * (M + 1) + 8 * 8, "ms_per_step": ms2 / args.steps}
    solve_info = None
    if args.solve:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = solver.solve(b_dev, k=3000, restart=M, tol=1e-12, gs_iters=args.gs, x_out=x_dev, want_H=False)
        torch.cuda.synchronize()
        solve_info = {"iters": r["iters"], "cycles": r["cycles"], "term": r["term"],
                      "true_relres": r["true_relres"], "wall_s": time.perf_counter() - t0}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_ours(prob)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "ms_per_step_median": ms_median,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, workloads/)",
            "config": bench_config(args.gs, world),
            "achieved_gbs_per_iteration_model": gbs_iter,
            "roofline_frac_iteration": gbs_iter / (peak * world),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src},
            "kernels": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                            "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 and v["bytes"] > 0 else None}
                        for k, v in ks.items() if v["launches"]},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if solve_info:
            line["solve_to_1e-12"] = solve_info
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
