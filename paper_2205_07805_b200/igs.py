"""Thin ctypes binding of libigs (include/igs.h): argument marshalling only.

Every step of the solve runs in the CUDA kernels of libigs.so; there is no CPU fallback —
if the library is missing or no CUDA device is visible, calls raise IgsError.
torch is used only for device memory (tensors' data_ptr), the current stream, and
torch.distributed to broadcast the NCCL unique id.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libigs.so")

IGS_OK, IGS_ERR_ARG, IGS_ERR_CUDA, IGS_ERR_NCCL, IGS_ERR_OOM, IGS_ERR_NONFINITE, IGS_ERR_STATE = range(7)
IGS_MEM_HOST, IGS_MEM_DEVICE = 0, 1
TERM = {0: "converged", 1: "maxiter", 2: "breakdown"}
KERNEL_KINDS = ["spmv", "block_dot", "allreduce", "small", "update", "halo", "cycle", "persist"]
STATUS_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_CUDA", 3: "ERR_NCCL", 4: "ERR_OOM",
                5: "ERR_NONFINITE", 6: "ERR_STATE"}

# every symbol include/igs.h declares
EXPORTS = ["igs_create", "igs_nccl_unique_id", "igs_workspace_bytes", "igs_bind_workspace",
           "igs_solve", "igs_solve_alg", "igs_stats", "igs_set_timing", "igs_kernel_stats", "igs_destroy",
           "igs_last_error", "igs_op_block_dot", "igs_op_spmv", "igs_op_update",
           "igs_op_trisolve", "igs_plan_ghosts", "igs_plan_remap", "igs_qr",
           "igs_op_basis_diag", "igs_bench_block_dot", "igs_set_timeout", "igs_create_virtual",
           "igs_virtual_spmv", "igs_virtual_solve", "igs_info", "igs_bench_update", "igs_plan_sell"]


class IgsError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class igs_result(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("H", ctypes.c_void_p), ("res_hist", ctypes.c_void_p),
                ("want_loo", ctypes.c_int), ("loo_frob", ctypes.c_double), ("iters", ctypes.c_int),
                ("cycles", ctypes.c_int), ("term", ctypes.c_int), ("true_relres", ctypes.c_double),
                ("h_cols", ctypes.c_int), ("basis_cols", ctypes.c_int), ("allreduces", ctypes.c_int64),
                ("reductions", ctypes.c_int64), ("lnorm_hist", ctypes.c_void_p),
                ("want_basis_diag", ctypes.c_int), ("s_norm", ctypes.c_double),
                ("sigma_min", ctypes.c_double), ("lgram_frob", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libigs.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise IgsError(IGS_ERR_STATE, "load", f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I, D, S = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        sig = {
            "igs_create": [ctypes.POINTER(P), I64, I64, I64, P, P, I, P, I64, I, I, P, I, I, P],
            "igs_nccl_unique_id": [P],
            "igs_workspace_bytes": [P, I],
            "igs_bind_workspace": [P, P, S],
            "igs_solve": [P, I, P, P, I, I, D, I, ctypes.POINTER(igs_result)],
            "igs_solve_alg": [P, I, P, P, I, I, D, I, ctypes.POINTER(igs_result)],
            "igs_stats": [P, P, P, P],
            "igs_set_timing": [P, I],
            "igs_set_timeout": [P, D],
            "igs_info": [P, I, P],
            "igs_create_virtual": [P, I, I64, P, P, P, I, P, I, P],
            "igs_virtual_spmv": [P, I, P, P, P],
            "igs_virtual_solve": [P, I, P, I, I, D, I, P],
            "igs_kernel_stats": [P, I, P, P, P],
            "igs_destroy": [P],
            "igs_last_error": [],
            "igs_op_block_dot": [I64, I, P, I64, P, P, P, P],
            "igs_op_spmv": [P, P, P],
            "igs_bench_block_dot": [I64, I, P, I64, P, P, P, I, P, P],
            "igs_bench_update": [I64, I, P, I64, P, P, P, P, D, P, P, I, P, P],
            "igs_op_update": [I64, I, P, I64, P, P, P, P, D, P, P, P],
            "igs_op_trisolve": [I, P, I, P, P, P],
            "igs_qr": [I64, I, P, I64, P, I64, P, I, P, P],
            "igs_op_basis_diag": [I64, I, P, I64, P, P],
            "igs_plan_ghosts": [I64, I64, P, P, I, I, P, P, P, P],
            "igs_plan_remap": [I64, I64, P, P, I, I64, P, P],
            "igs_plan_sell": [I64, P, P, P, I, I64, P, P, P, P, P, P, I64, P, I64, P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.igs_workspace_bytes.restype = ctypes.c_size_t
        L.igs_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != IGS_OK:
        raise IgsError(st, where, lib().igs_last_error().decode(errors="replace"))


def _ptr(a) -> Optional[int]:
    """data pointer of a torch tensor or numpy array (None passes NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------------- C-ABI names
def igs_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().igs_nccl_unique_id(buf), "igs_nccl_unique_id")
    return buf.raw


def igs_create(n_global, row_begin, n_local, rowptr, colind, values, *, where=IGS_MEM_HOST,
               cuda_device=0, nccl_unique_id: Optional[bytes] = None, rank=0, nranks=1,
               stream=None) -> int:
    h = ctypes.c_void_p()
    bits = 64 if colind.dtype.itemsize == 8 else 32
    uid = ctypes.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id else None
    nnz = int(values.numel() if hasattr(values, "numel") else values.size)
    _check(lib().igs_create(ctypes.byref(h), int(n_global), int(row_begin), int(n_local),
                            _ptr(rowptr), _ptr(colind), bits, _ptr(values), nnz, where,
                            int(cuda_device), uid, int(rank), int(nranks), _stream_ptr(stream)),
           "igs_create")
    return h.value


def igs_destroy(ctx: int):
    _check(lib().igs_destroy(ctx), "igs_destroy")


def igs_solve(ctx: int, vec_mem: int, b, x0, k: int, restart: int, tol: float, gs_iters: int,
              res: igs_result):
    _check(lib().igs_solve(ctx, vec_mem, _ptr(b), _ptr(x0), int(k), int(restart), float(tol),
                           int(gs_iters), ctypes.byref(res)), "igs_solve")


ALGORITHMS = {"igs1": 1, "igs2": 2, "alg3": 2, "igs2_two": 3, "mgs": 4}


def igs_solve_alg(ctx: int, vec_mem: int, b, x0, k: int, restart: int, tol: float, algorithm: int,
                  res: igs_result):
    _check(lib().igs_solve_alg(ctx, vec_mem, _ptr(b), _ptr(x0), int(k), int(restart), float(tol),
                               int(algorithm), ctypes.byref(res)), "igs_solve_alg")


def igs_stats(ctx: int) -> dict:
    a, h, it = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().igs_stats(ctx, ctypes.byref(a), ctypes.byref(h), ctypes.byref(it)), "igs_stats")
    return {"allreduces": a.value, "halo_msgs": h.value, "iterations": it.value}


def igs_set_timing(ctx: int, on: int):
    _check(lib().igs_set_timing(ctx, int(on)), "igs_set_timing")


def igs_kernel_stats(ctx: int) -> dict:
    out = {}
    for kind, name in enumerate(KERNEL_KINDS):
        ms, n, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _check(lib().igs_kernel_stats(ctx, kind, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by)),
               "igs_kernel_stats")
        out[name] = {"ms": ms.value, "launches": n.value, "bytes": by.value}
    return out


def igs_workspace_bytes(ctx: int, max_restart: int) -> int:
    return int(lib().igs_workspace_bytes(ctx, int(max_restart)))


def igs_bind_workspace(ctx: int, dev_ptr: int, nbytes: int):
    _check(lib().igs_bind_workspace(ctx, dev_ptr, int(nbytes)), "igs_bind_workspace")


def igs_op_block_dot(n, p, V, ld, u, z, out, stream=None):
    _check(lib().igs_op_block_dot(int(n), int(p), _ptr(V), int(ld), _ptr(u), _ptr(z), _ptr(out),
                                  _stream_ptr(stream)), "igs_op_block_dot")


def igs_bench_block_dot(n, p, V, ld, u, z, out, reps=10, stream=None) -> float:
    """Mean milliseconds per block-dot launch over `reps` back-to-back launches (CUDA events)."""
    ms = ctypes.c_float(0.0)
    _check(lib().igs_bench_block_dot(int(n), int(p), _ptr(V), int(ld), _ptr(u), _ptr(z), _ptr(out), int(reps),
                                     ctypes.byref(ms), _stream_ptr(stream)), "igs_bench_block_dot")
    return ms.value


def igs_bench_update(n, p, V, ld, u, z, alpha, beta, gamma, v_out, u_next, reps=10, stream=None) -> float:
    """Mean milliseconds per fused-update launch over `reps` back-to-back launches."""
    ms = ctypes.c_float(0.0)
    _check(lib().igs_bench_update(int(n), int(p), _ptr(V), int(ld), _ptr(u), _ptr(z), _ptr(alpha), _ptr(beta),
                                  float(gamma), _ptr(v_out), _ptr(u_next), int(reps), ctypes.byref(ms),
                                  _stream_ptr(stream)), "igs_bench_update")
    return ms.value


def igs_op_spmv(ctx: int, x, y):
    _check(lib().igs_op_spmv(ctx, _ptr(x), _ptr(y)), "igs_op_spmv")


def igs_op_update(n, p, V, ld, u, z, alpha, beta, gamma, v_out, u_next, stream=None):
    _check(lib().igs_op_update(int(n), int(p), _ptr(V), int(ld), _ptr(u), _ptr(z), _ptr(alpha),
                               _ptr(beta), float(gamma), _ptr(v_out), _ptr(u_next),
                               _stream_ptr(stream)), "igs_op_update")


def igs_op_basis_diag(n, c, V, ld, stream=None):
    """[||I - V^T V||_F, ||S||_2, sigma_min(V)] of a device block V (n x c, col-major)."""
    out = np.zeros(3)
    _check(lib().igs_op_basis_diag(int(n), int(c), _ptr(V), int(ld), out.ctypes.data, _stream_ptr(stream)),
           "igs_op_basis_diag")
    return out


def igs_qr(n, m, A, lda, Q, ldq, R, sweeps=2, stream=None) -> int:
    """Algorithm 1 QR on the device (device tensors); returns the number of reductions."""
    red = ctypes.c_int64(0)
    _check(lib().igs_qr(int(n), int(m), _ptr(A), int(lda), _ptr(Q), int(ldq), _ptr(R), int(sweeps),
                        ctypes.byref(red), _stream_ptr(stream)), "igs_qr")
    return red.value


def igs_op_trisolve(order, L, ldl, b, x, stream=None):
    _check(lib().igs_op_trisolve(int(order), _ptr(L), int(ldl), _ptr(b), _ptr(x),
                                 _stream_ptr(stream)), "igs_op_trisolve")


def igs_plan_ghosts(row_begin, n_local, rowptr, colind, nranks, bounds):
    """Host-only: (ghosts int64[], ghost_owner_count int64[nranks])."""
    bits = 64 if colind.dtype.itemsize == 8 else 32
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    cnt = np.zeros(nranks, dtype=np.int64)
    ng = ctypes.c_int64(0)
    _check(lib().igs_plan_ghosts(int(row_begin), int(n_local), _ptr(rowptr), _ptr(colind), bits,
                                 int(nranks), _ptr(bounds), ctypes.byref(ng), None, _ptr(cnt)),
           "igs_plan_ghosts")
    ghosts = np.zeros(max(ng.value, 1), dtype=np.int64)
    _check(lib().igs_plan_ghosts(int(row_begin), int(n_local), _ptr(rowptr), _ptr(colind), bits,
                                 int(nranks), _ptr(bounds), ctypes.byref(ng), _ptr(ghosts), _ptr(cnt)),
           "igs_plan_ghosts")
    return ghosts[:ng.value], cnt


def igs_plan_remap(row_begin, n_local, rowptr, colind, ghosts):
    bits = 64 if colind.dtype.itemsize == 8 else 32
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    ghosts = np.ascontiguousarray(ghosts, dtype=np.int64)
    out = np.zeros(max(int(rowptr[-1]), 1), dtype=np.int64)
    _check(lib().igs_plan_remap(int(row_begin), int(n_local), _ptr(rowptr), _ptr(colind), bits,
                                int(ghosts.size), _ptr(ghosts) if ghosts.size else None, _ptr(out)),
           "igs_plan_remap")
    return out[:int(rowptr[-1])]


def igs_plan_sell(n, rowptr, local_col, values, want_diag=True, bnd_rows=()):
    """The SELL-32 arrays igs_create builds (host only): dict with ptr, cptr, diag, len, mask,
    val, col, n_diag -- or None when a row has >= 255 entries (no SELL copy)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    local_col = np.ascontiguousarray(local_col, dtype=np.int64)
    values = np.ascontiguousarray(values, dtype=np.float64)
    bnd = np.ascontiguousarray(bnd_rows, dtype=np.int64)
    ns = (int(n) + 31) // 32
    nv, nc, nd = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    out = {"ptr": np.zeros(ns + 1, np.int64), "cptr": np.zeros(ns + 1, np.int64),
           "diag": np.zeros(8 * ns, np.int32), "len": np.zeros(32 * ns, np.uint8),
           "mask": np.zeros(32 * ns, np.uint8)}

    def call(val, col):
        _check(lib().igs_plan_sell(int(n), _ptr(rowptr), _ptr(local_col) if local_col.size else None,
                                   _ptr(values) if values.size else None, int(bool(want_diag)),
                                   int(bnd.size), _ptr(bnd) if bnd.size else None,
                                   _ptr(out["ptr"]), _ptr(out["cptr"]), _ptr(out["diag"]) if ns else None,
                                   _ptr(out["len"]) if ns else None, _ptr(out["mask"]) if ns else None,
                                   0 if val is None else int(val.size), None if val is None else _ptr(val),
                                   0 if col is None else int(col.size), None if col is None else _ptr(col),
                                   ctypes.byref(nv), ctypes.byref(nc), ctypes.byref(nd)), "igs_plan_sell")

    call(None, None)
    if nv.value < 0:
        return None
    out["val"] = np.zeros(max(nv.value, 1), np.float64)
    out["col"] = np.zeros(max(nc.value, 1), np.int64)
    call(out["val"], out["col"])
    out["val"], out["col"] = out["val"][:nv.value], out["col"][:nc.value]
    out["n_diag"] = nd.value
    return out


# ------------------------------------------------------------------------- convenience
INFO_KEYS = ["xchg", "nranks", "n_ghost", "n_send", "n_peers", "n_bnd", "graph_launches", "pcycle_launches",
             "sell", "csr_compact", "sell_diag_slices", "sell_walk", "spmv_bytes", "pcycle_ares"]


def igs_info(ctx: int) -> dict:
    out = {}
    for i, k in enumerate(INFO_KEYS):
        v = ctypes.c_int64(0)
        _check(lib().igs_info(ctx, i, ctypes.byref(v)), "igs_info")
        out[k] = v.value
    return out


def igs_set_timeout(ctx: int, seconds: float):
    _check(lib().igs_set_timeout(ctx, float(seconds)), "igs_set_timeout")


class VirtualGroup:
    """G virtual-rank contexts of one global CSR on one device (igs_create_virtual): the
    G > 1 halo path of the SpMV (pack kernel, ghost copies, interior/boundary split) on a
    single GPU.  Test hook; `spmv(xs, ys[, bs])` takes per-rank device tensors."""

    def __init__(self, csr, bounds, *, device: int = 0, stream=None):
        import torch
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        self.G = len(self.bounds) - 1
        rowptr = np.ascontiguousarray(csr.rowptr, dtype=np.int64)
        colind = np.ascontiguousarray(csr.colind)
        values = np.ascontiguousarray(csr.values, dtype=np.float64)
        bits = 64 if colind.dtype.itemsize == 8 else 32
        arr = (ctypes.c_void_p * self.G)()
        _check(lib().igs_create_virtual(arr, self.G, int(csr.n_cols), self.bounds.ctypes.data, rowptr.ctypes.data,
                                        colind.ctypes.data, bits, values.ctypes.data, int(device),
                                        _stream_ptr(self.stream)), "igs_create_virtual")
        self.ctxs = [arr[i] for i in range(self.G)]
        self._arr = arr

    def spmv(self, xs, ys, bs=None):
        G = self.G
        px = (ctypes.c_void_p * G)(*[_ptr(t) for t in xs])
        py = (ctypes.c_void_p * G)(*[_ptr(t) for t in ys])
        pb = (ctypes.c_void_p * G)(*[_ptr(t) for t in bs]) if bs is not None else None
        _check(lib().igs_virtual_spmv(self._arr, G, px, py, pb), "igs_virtual_spmv")

    def solve(self, bs, xs, *, k: int, restart: int = 0, tol: float = 0.0, algorithm: str = "igs2",
              want_loo: bool = False) -> list:
        """All members' igs_solve_alg at once (igs_virtual_solve): bs / xs are per-rank device
        tensors (rank r's rows); returns one result dict per member (H replicated)."""
        G = self.G
        m1 = restart if 0 < restart < k else k
        res = (igs_result * G)()
        keep = []
        for r in range(G):
            H = np.zeros((m1 + 1) * m1)
            rh = np.full(k + 1, np.nan)
            lh = np.full(k + 1, np.nan)
            keep.append((H, rh, lh))
            res[r].x = _ptr(xs[r])
            res[r].H = H.ctypes.data
            res[r].res_hist = rh.ctypes.data
            res[r].lnorm_hist = lh.ctypes.data
            res[r].want_loo = int(want_loo)
        pb = (ctypes.c_void_p * G)(*[_ptr(t) for t in bs])
        _check(lib().igs_virtual_solve(self._arr, G, pb, int(k), int(restart), float(tol),
                                       ALGORITHMS[algorithm], res), "igs_virtual_solve")
        out = []
        for r in range(G):
            H, rh, lh = keep[r]
            q = res[r]
            out.append(dict(iters=q.iters, cycles=q.cycles, term=TERM[q.term], true_relres=q.true_relres,
                            loo=q.loo_frob, h_cols=q.h_cols, basis_cols=q.basis_cols,
                            allreduces=q.allreduces, reductions=q.reductions,
                            res_hist=rh[:q.iters + 1], H=H.reshape(m1, m1 + 1).T, m=m1))
        return out

    def stats(self) -> list:
        return [igs_stats(c) for c in self.ctxs]

    def close(self):
        for c in getattr(self, "ctxs", []) or []:
            if c:
                igs_destroy(c)
        self.ctxs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """One rank's IGS-GMRES solver: `Solver(csr, ...)` then `.solve(b, k=..., ...)`.

    csr: object with n_rows, n_cols, row_begin, rowptr, colind, values (numpy, host) --
    e.g. workloads.Csr.  For nranks > 1 pass nccl_unique_id (bytes from rank 0's
    igs_nccl_unique_id(), broadcast by the caller) and this rank's row block.
    """

    def __init__(self, csr, *, device: int = 0, stream=None, rank: int = 0, nranks: int = 1,
                 nccl_unique_id: Optional[bytes] = None):
        import torch
        torch.cuda.set_device(device)
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.n_local = int(csr.n_rows)
        self.n_global = int(csr.n_cols)
        self.row_begin = int(csr.row_begin)
        self.nranks = nranks
        rowptr = np.ascontiguousarray(csr.rowptr, dtype=np.int64)
        colind = np.ascontiguousarray(csr.colind)
        values = np.ascontiguousarray(csr.values, dtype=np.float64)
        self.ctx = igs_create(self.n_global, self.row_begin, self.n_local, rowptr, colind, values,
                              where=IGS_MEM_HOST, cuda_device=device, nccl_unique_id=nccl_unique_id,
                              rank=rank, nranks=nranks, stream=self.stream)

    def close(self):
        if getattr(self, "ctx", None):
            igs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, b, *, k: int, restart: int = 0, tol: float = 0.0, gs_iters: int = 2,
              x0=None, x_out=None, want_loo: bool = False, want_H: bool = True,
              algorithm: Optional[str] = None, want_diag: bool = False) -> dict:
        """b/x0/x_out: torch CUDA tensors (IGS_MEM_DEVICE) or host arrays/tensors
        (IGS_MEM_HOST: the H2D/D2H copies happen inside the call).  algorithm in
        {'igs1','igs2','igs2_two','mgs'} overrides gs_iters (igs_solve_alg)."""
        import torch
        dev = isinstance(b, torch.Tensor) and b.is_cuda
        if x_out is None:
            x_out = (torch.empty(self.n_local, dtype=torch.float64, device=b.device) if dev
                     else np.empty(self.n_local))
        m1 = restart if 0 < restart < k else k
        H = np.zeros((m1 + 1) * m1) if want_H else None
        rh = np.full(k + 1, np.nan)
        lh = np.full(k + 1, np.nan)
        res = igs_result()
        res.lnorm_hist = lh.ctypes.data
        res.x = _ptr(x_out)
        res.H = _ptr(H)
        res.res_hist = rh.ctypes.data
        res.want_loo = int(want_loo)
        res.want_basis_diag = int(want_diag)
        if algorithm is None:
            igs_solve(self.ctx, IGS_MEM_DEVICE if dev else IGS_MEM_HOST, b, x0, k, restart, tol,
                      gs_iters, res)
        else:
            igs_solve_alg(self.ctx, IGS_MEM_DEVICE if dev else IGS_MEM_HOST, b, x0, k, restart, tol,
                          ALGORITHMS[algorithm], res)
        out = dict(x=x_out, iters=res.iters, cycles=res.cycles, term=TERM[res.term],
                   true_relres=res.true_relres, loo=res.loo_frob, h_cols=res.h_cols,
                   basis_cols=res.basis_cols, allreduces=res.allreduces, reductions=res.reductions,
                   res_hist=rh[:res.iters + 1], lnorm_hist=lh[:res.iters + 1], m=m1,
                   s_norm=res.s_norm, sigma_min=res.sigma_min, lgram=res.lgram_frob)
        if want_H:
            out["H"] = H.reshape(m1, m1 + 1).T
        return out

    def spmv(self, x, y):
        igs_op_spmv(self.ctx, x, y)

    def set_timing(self, on: int):
        igs_set_timing(self.ctx, on)

    def set_timeout(self, seconds: float):
        igs_set_timeout(self.ctx, seconds)

    def info(self) -> dict:
        return igs_info(self.ctx)

    def kernel_stats(self) -> dict:
        return igs_kernel_stats(self.ctx)

    def stats(self) -> dict:
        return igs_stats(self.ctx)
