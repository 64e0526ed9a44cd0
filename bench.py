#!/usr/bin/env python3
"""bench.py -- Arnoldi iterations/s and achieved HBM GB/s of the IGS-GMRES hot path on B200.

Workload (BASELINE.json configs[3], "c4"): 3D convection-diffusion 7-point stencil on a
256^3 grid (n = 16,777,216, nnz = 117,047,296, CSR FP64, int32 columns), convection
(100,50,25), b ~ U(0,1) seed 3, x0 = 0, GMRES(100).  One "step" = one restart cycle of 100
Arnoldi iterations through igs_solve (k = restart = 100, tol = 0, gs_iters = 2 = Alg. 3):
||b||, r0, priming, 100 x [SpMV, fused block dot, (cross-rank sum), small step, fused
update], least squares, x += V y, final residual.  value = Arnoldi iterations (all ranks' one
shared Krylov process) per second, measured with per-launch timing OFF (the production
path); the per-kernel split comes from a second, instrumented pass.  The basis V (13.6 GB)
is far larger than L2, so no flush is needed between steps.  N > 1: the same 256^3 problem
row-block sharded over N ranks (strong scaling): z-slabs, halo send/recv of one plane per
neighbour, one cross-rank reduction of 2(p+1) doubles per iteration (fused into the block
dot over NVLink by default, else ncclAllReduce).  The line also carries the c4 solve as
specified (GMRES(100) to a true relative residual of 1e-12) next to the oracle's committed
record (tests/golden/oracle_c4_gs2.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dry-run]

--gpus N without WORLD_SIZE in the environment re-launches itself through
torch.distributed.run with N processes (one per GPU); under torchrun WORLD_SIZE must equal N.
--dry-run forms the process group (gloo, no GPU work) and prints the ranks it formed.
--impl reference times the CPU oracle (oracle/, plain FP64 C + OpenMP) on the host cores,
rank 0 only; each step is a bounded sample (the first 50 Arnoldi iterations of the same
cycle), projected to the cycle-average iteration with the byte model of DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
CPU_SAMPLE_ITERS = 50       # oracle sample: iterations 1..50 of the cycle (~12 s on 16 cores)
CPU_SAMPLE_ITERS_1T = 12    # the same at one thread: iterations 1..12 (~8 s)
NOMINAL_HBM_GBS = 8000.0    # north-star denominator (B200 HBM3e, nominal)


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


# --------------------------------------------------------------------- process launch
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard_bounds(n, world, rank):
    """Rank `rank`'s contiguous row block of the N_GRID^3 grid: whole z-planes."""
    plane = N_GRID * N_GRID
    return (N_GRID * rank // world) * plane, (N_GRID * (rank + 1) // world) * plane


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(nproc: int) -> int:
    """--gpus N without a launcher: start N ranks through torch.distributed.run (one process
    per GPU, rendezvous on 127.0.0.1) running this script with the same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {nproc} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def dry_run(args, rank, world) -> int:
    """Form the process group the bench would use (gloo here: no GPU work) and report it."""
    import torch.distributed as dist
    dist.init_process_group("gloo")
    got = [None] * world
    dist.all_gather_object(got, {"rank": rank, "world": int(os.environ.get("WORLD_SIZE", "1")),
                                 "local_rank": int(os.environ.get("LOCAL_RANK", "0")), "pid": os.getpid()})
    if rank == 0:
        print(json.dumps({"dry_run": True, "gpus": args.gpus, "world": world, "ranks": got}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------- reference arm / CPU
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


def oracle_sample(iters: int, gs: int) -> dict:
    """Time the oracle on the first `iters` Arnoldi iterations of the c4 GMRES(100) cycle
    (this process; OMP_NUM_THREADS decides the cores).  Returns it/s projected to the cycle
    average by the byte model, and the raw numbers."""
    import oracle
    import workloads as W
    prob = W.config("c4")
    A, b = prob.A, prob.b
    n, nnz = A.n_rows, A.nnz
    oracle.build()
    t0 = time.perf_counter()
    o = oracle.gmres(A, b, iters, restart=M, tol=0.0, variant="igs2" if gs == 2 else "igs1", dot_block=4096)
    t = time.perf_counter() - t0
    assert o["iters"] == iters
    sample_bytes = sum(byte_model(n, nnz, p) for p in range(1, iters + 1))
    gbs = sample_bytes / t / 1e9
    return {"value": gbs * 1e9 / cycle_avg_bytes(n, nnz), "unit": UNIT, "cores": oracle.num_threads(),
            "kind": "oracle", "wall_s": t, "raw_it_s": iters / t, "gbs": gbs,
            "sample": (f"first {iters} iterations of one c4 GMRES(100) cycle (gs_iters={gs}, blocked FP64 "
                       f"dots), {t:.1f} s wall; projected to the cycle-average iteration by the byte model "
                       f"({iters / t:.3f} it/s raw, {gbs:.1f} GB/s)"), **host_cpu()}


def cpu_baseline_subprocess(gs: int, iters: int, threads: int | None) -> dict | None:
    """The oracle timed in a child process (keeps the GPU arm's process free of the oracle
    library); threads = None: all host cores."""
    env = dict(os.environ)
    if threads:
        env["OMP_NUM_THREADS"] = str(threads)
    code = ("import json,sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench.oracle_sample(%d, %d)))" % (ROOT, iters, gs))
    try:
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle, rank 0 only (the other ranks exit 0)."""
    if rank != 0:
        return 0
    times, last = [], None
    for i in range(args.warmup + args.steps):
        s = oracle_sample(CPU_SAMPLE_ITERS, args.gs)
        if i >= args.warmup:
            times.append(s["wall_s"])
            last = s
    t = float(np.mean(times))
    val = last["value"] * last["wall_s"] / t
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, workloads/)",
            "config": bench_config(args.gs, world),
            "cpu_baseline": {**last, "value": val},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ the GPU arm
def golden_c4(gs: int) -> dict | None:
    path = os.path.join(ROOT, "tests", "golden", f"oracle_c4_gs{gs}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return None


def halo_plan_bytes(prob, world, rank, r0, r1) -> dict:
    """Ghost entries this rank receives / sends per SpMV (the library's own planner)."""
    import paper_2205_07805_b200 as P
    if world == 1:
        return {"recv": 0, "send": 0}
    plane = N_GRID * N_GRID
    bounds = np.array([(N_GRID * q // world) * plane for q in range(world + 1)], dtype=np.int64)
    g, _ = P.igs_plan_ghosts(r0, r1 - r0, prob.A.rowptr, prob.A.colind, world, bounds)
    return {"recv": int(len(g))}


def run_ours(args, rank, world, local) -> int:
    import torch
    import torch.distributed as dist

    import paper_2205_07805_b200 as P
    import workloads as W

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_global = N_GRID ** 3
    r0, r1 = shard_bounds(n_global, world, rank)
    prob = W.config("c4", row_begin=r0, row_end=r1)
    stream = torch.cuda.current_stream()

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

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def all_ok(flag: bool) -> bool:
        if world == 1:
            return flag
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def make_solver():
        uid = None
        if world > 1:
            obj = [P.igs_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return P.Solver(prob.A, device=local, stream=stream, rank=rank, nranks=world, nccl_unique_id=uid)

    solver = make_solver()
    n_loc = prob.A.n_rows
    b_dev = torch.from_numpy(prob.b).cuda()
    x_dev = torch.empty(n_loc, dtype=torch.float64, device="cuda")

    def step_dev():
        return solver.solve(b_dev, k=M, restart=M, tol=0.0, gs_iters=args.gs, x_out=x_dev, want_H=False)

    # ---- preflight (N > 1): the first cycle runs the collective path end to end; if any rank
    # fails (e.g. the fused NVLink exchange times out), every rank rebuilds on ncclAllReduce
    path_note = None
    if world > 1:
        # a peer that never arrives at the fused exchange's barrier fails the preflight in
        # seconds (device bound 20 s, host deadline 40 s), not after the 120 s default
        solver.set_timeout(20.0)
    try:
        r = step_dev()
        ok = r["iters"] == M
    except P.IgsError as e:
        ok, path_note = False, str(e)[:300]
        print(f"[bench rank {rank}] preflight failed: {e}", file=sys.stderr, flush=True)
    if not all_ok(ok):
        if world == 1:
            raise RuntimeError(f"preflight solve failed: {path_note}")
        try:
            solver.close()
        except Exception:
            pass
        os.environ["IGS_XCHG"] = "0"
        solver = make_solver()
        path_note = path_note or "a peer rank failed the preflight"
        r = step_dev()
        assert r["iters"] == M, r
    if world > 1:
        solver.set_timeout(120.0)
    info = solver.info()
    # replicated k x k state must be bit-identical on every rank
    replicated_ok = None
    if world > 1:
        h = torch.from_numpy(np.ascontiguousarray(r["res_hist"])).cuda()
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        replicated_ok = all(bool(torch.equal(hs[0], t)) for t in hs)
    for _ in range(max(0, args.warmup - 1)):
        r = step_dev()
        assert r["iters"] == M, r

    # ---------------- timed region: production path (per-launch timing off) ---------------
    clocks = ClockSampler(local)
    solver.set_timing(0)
    barrier()
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    iters = 0
    for i in range(args.steps):
        iters += step_dev()["iters"]
        ev[i + 1].record(stream)
    ev[-1].synchronize()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(ev[0].elapsed_time(ev[-1]))
    step_ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    ms_median = max_over_ranks(step_ms[len(step_ms) // 2])
    value = iters / (ms / 1e3)

    # ---------------- per-kernel split: a second, instrumented pass --------------------------
    ksteps = max(2, min(args.steps, 5))
    solver.set_timing(2)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(ksteps):
        step_dev()
    f1.record(stream)
    f1.synchronize()
    ms_instr = max_over_ranks(f0.elapsed_time(f1)) / ksteps
    ks = solver.kernel_stats()
    solver.set_timing(0)
    nnz_g = 7 * N_GRID ** 3 - 6 * N_GRID ** 2
    model_bytes = args.steps * sum(byte_model(n_global, nnz_g, p) for p in range(1, M + 1))
    gbs_iter = model_bytes / (ms / 1e3) / 1e9
    # the same sum with the SpMV's stored-format bytes (SELL-32 with diagonal slices streams
    # less than the CSR definition the model fixes): what the iteration actually moves, V twice
    spmv_moved = sum_over_ranks(float(info["spmv_bytes"]))
    moved_bytes = args.steps * sum(spmv_moved + 16.0 * n_global * p for p in range(1, M + 1))
    gbs_iter_moved = moved_bytes / (ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    # dominant kernel (largest device time) and its achieved algorithmic GB/s (this rank's
    # bytes over its own launches; rank 0's split)
    dom = max((k for k in ks if ks[k]["launches"] > 0), key=lambda k: ks[k]["ms"])
    dk = ks[dom]
    achieved = dk["bytes"] / (dk["ms"] / 1e3) / 1e9 if dk["ms"] > 0 else 0.0
    launches_per_step = sum(v["launches"] for v in ks.values() if v["launches"]) / ksteps
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

    # ---------------- end-to-end: host buffers, H2D/D2H inside the timed region -------------
    e2e = None
    if not args.no_e2e:
        b_host = torch.from_numpy(prob.b).pin_memory()
        x_host = torch.empty(n_loc, dtype=torch.float64).pin_memory()
        solver.solve(b_host, k=M, restart=M, tol=0.0, gs_iters=args.gs, x_out=x_host, want_H=False)
        barrier()
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

    # ---------------- c4 as specified: GMRES(100) to 1e-12, next to the oracle's record ------
    solve_info = None
    if not args.no_solve:
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        rs = solver.solve(b_dev, k=3000, restart=M, tol=1e-12, gs_iters=args.gs, x_out=x_dev, want_H=False)
        g1.record(stream)
        g1.synchronize()
        tms = max_over_ranks(g0.elapsed_time(g1))
        solve_info = {"iters": rs["iters"], "cycles": rs["cycles"], "term": rs["term"],
                      "true_relres": rs["true_relres"], "device_s": tms / 1e3,
                      "it_s": rs["iters"] / (tms / 1e3)}
        gold = golden_c4(args.gs)
        if gold:
            solve_info["oracle"] = {k: gold[k] for k in ("iters", "cycles", "term", "true_relres", "beta")}
            solve_info["oracle"]["record"] = f"tests/golden/oracle_c4_gs{args.gs}.json"
            if world == 1:  # beta(x) with the oracle's ||A||_2 (shared, reading R11)
                import oracle
                xg = x_dev.cpu().numpy()
                solve_info["beta"] = oracle.backward_error(prob.A, prob.b, xg, gold["normA_2"])
    cpu = cpu1 = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_subprocess(args.gs, CPU_SAMPLE_ITERS, None)
        cpu1 = cpu_baseline_subprocess(args.gs, CPU_SAMPLE_ITERS_1T, 1)
        if cpu and "value" in cpu:
            cpu["one_thread"] = cpu1
    halo = halo_plan_bytes(prob, world, rank, r0, r1)
    halo_all = [halo["recv"]]
    if world > 1:
        got = [None] * world
        dist.all_gather_object(got, halo["recv"])
        halo_all = got
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
            "roofline_frac_iteration_nominal_8tbs": gbs_iter / (NOMINAL_HBM_GBS * world),
            "achieved_gbs_per_iteration_moved": gbs_iter_moved,
            "roofline_frac_iteration_moved": gbs_iter_moved / (peak * world),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src, "frac_nominal_8tbs": achieved / NOMINAL_HBM_GBS},
            "kernels": {k: {"ms_per_step": v["ms"] / ksteps, "launches_per_step": v["launches"] / ksteps,
                            "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 and v["bytes"] > 0 else None,
                            # the SpMV's "gbs" is the CSR byte model; the stored format
                            # (SELL-32 with diagonal slices) streams fewer bytes -- those are gbs_moved
                            **({"gbs_moved": info["spmv_bytes"] * v["launches"] / (v["ms"] / 1e3) / 1e9}
                               if k == "spmv" and v["ms"] > 0 else {})}
                        for k, v in ks.items() if v["launches"]},
            "kernel_split_pass": {"steps": ksteps, "ms_per_step": ms_instr,
                                  "note": "CUDA events around every launch (instrumented); value is the uninstrumented pass"},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "multi_gpu": {"ranks": world,
                          "reduction_path": ("fused NVLink exchange (NCCL symmetric window, in the block dot)"
                                             if info["xchg"] else ("ncclAllReduce" if world > 1 else "none (1 rank)")),
                          "fallback_reason": path_note,
                          "halo_bytes_per_iteration": 8 * int(sum(halo_all)),
                          "halo_entries_per_rank": halo_all,
                          "replicated_state_bitwise_identical": replicated_ok,
                          "graph_replayed_cycles": info["graph_launches"]},
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gs", type=int, default=2, choices=[1, 2])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the full c4 solve to 1e-12")
    ap.add_argument("--dry-run", action="store_true", help="form the process group only (gloo)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1 and (args.impl == "ours" or args.dry_run):
        return relaunch(args.gpus)
    rank, world, local = dist_env()
    if launched and world != args.gpus:
        print(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}: refusing to run a different "
              f"number of ranks than requested", file=sys.stderr, flush=True)
        return 2
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world if launched else args.gpus)
    try:
        return run_ours(args, rank, world, local)
    except Exception as e:
        # a failed rank must not hang the job: report and leave without collective teardown
        print(f"[bench rank {rank}] FAILED: {type(e).__name__}: {e}", file=sys.stderr, flush=True)
        sys.stderr.flush()
        sys.stdout.flush()
        os._exit(3)


if __name__ == "__main__":
    sys.exit(main())
