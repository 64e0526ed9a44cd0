"""CPU FP64 oracle for the IGS-GMRES hot path (arXiv 2205.07805).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this package.  It shares no code with
the CUDA path in paper_2205_07805_b200/ and never imports it.

`oracle.c` holds the algorithms (step by step in the paper's order); this module loads
it with ctypes and adds the numpy diagnostics of §1/§4/§5 of the paper (loss of
orthogonality, backward error, Arnoldi relation, kappa(B_k), ||S_k||).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MGS, IGS1, IGS2_TWO, IGS2_ONE = 0, 1, 2, 3
VARIANTS = {"mgs": MGS, "igs1": IGS1, "igs2_two": IGS2_TWO, "igs2": IGS2_ONE, "alg3": IGS2_ONE}
TERM = {0: "converged", 1: "maxiter", 2: "breakdown"}
EPS = np.finfo(np.float64).eps


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -O2 -fopenmp -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.oracle_gmres.restype = I
        _lib.oracle_gmres.argtypes = [I64, P, P, P, P, P, I, I, D, I, I64, P, P, P, P, P, P, P, P]
        _lib.oracle_spmv.restype = None
        _lib.oracle_spmv.argtypes = [I64, P, P, P, P, P]
        _lib.oracle_dot.restype = D
        _lib.oracle_dot.argtypes = [I64, P, P, I64]
        _lib.oracle_forward_solve_unit.restype = None
        _lib.oracle_forward_solve_unit.argtypes = [I, P, I, P, P]
        _lib.oracle_hessenberg_lsq.restype = D
        _lib.oracle_hessenberg_lsq.argtypes = [I, P, I, D, P]
        _lib.oracle_num_threads.restype = I
        _lib.oracle_igs_qr.restype = I
        _lib.oracle_igs_qr.argtypes = [I64, I, P, I64, I, I64, P, I64, P, P, P]
        _lib.oracle_gemv.restype = None
        _lib.oracle_gemv.argtypes = [I64, I, P, I64, P, P]
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _csr64(A):
    return (np.ascontiguousarray(A.rowptr, dtype=np.int64),
            np.ascontiguousarray(A.colind, dtype=np.int64),
            np.ascontiguousarray(A.values, dtype=np.float64))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ------------------------------------------------------------------ primitives
def spmv(A, x) -> np.ndarray:
    rp, ci, v = _csr64(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.n_rows)
    lib().oracle_spmv(A.n_rows, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def dot(a, b, block: int = 0) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().oracle_dot(a.size, _p(a), _p(b), int(block)))


def block_dot(Vp, u, z, block: int = 0) -> np.ndarray:
    """[V_p, u]^T [u, z] laid out as [V_p^T u (p), u.u, V_p^T z (p), u.z] — the single
    reduction of Alg. 3 Step 4 / Alg. 2 Steps 5-6."""
    p = Vp.shape[1]
    out = np.empty(2 * (p + 1))
    for j in range(p):
        out[j] = dot(Vp[:, j], u, block)
    out[p] = dot(u, u, block)
    for j in range(p):
        out[p + 1 + j] = dot(Vp[:, j], z, block)
    out[2 * p + 1] = dot(u, z, block)
    return out


def gemv(V, c) -> np.ndarray:
    """t = V c, each row summed over columns in natural order."""
    V = np.asfortranarray(V, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    t = np.empty(V.shape[0])
    lib().oracle_gemv(V.shape[0], V.shape[1], _p(V), V.shape[0], _p(c), _p(t))
    return t


def update(Vp, u, z, alpha, beta, gamma):
    """The fused update of Alg. 3 Steps 10-13, in the oracle's arithmetic:
    v = (u - V_p alpha) / gamma (alpha None: v = u / gamma, Alg. 2 Step 7);
    u' = z / gamma - (V_p beta[:p] + v beta[p])  (Step 13 as V_{p+1} r1)."""
    p = Vp.shape[1]
    w = u - gemv(Vp, alpha) if alpha is not None else u.copy()
    v = w / gamma
    if z is None:
        return v, None
    Vp1 = np.column_stack([Vp, v])
    return v, z / gamma - gemv(Vp1, beta[:p + 1])


def forward_solve_unit(L, b) -> np.ndarray:
    """(I + L)^{-1} b, L strictly lower (only the strictly lower part is read)."""
    L = np.asfortranarray(L, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    lib().oracle_forward_solve_unit(b.size, _p(L), L.shape[0], _p(b), _p(x))
    return x


def hessenberg_lsq(H, rho):
    """y = argmin ||rho e1 - H y|| by progressive Givens; returns (y, |g_p|)."""
    H = np.asfortranarray(H, dtype=np.float64)
    p = H.shape[1]
    y = np.empty(p)
    res = lib().oracle_hessenberg_lsq(p, _p(H), H.shape[0], float(rho), _p(y))
    return y, float(res)


# ------------------------------------------------------------------ the solver
def gmres(A, b, k: int, restart: int = 0, tol: float = 0.0, variant="igs2", x0=None,
          dot_block: int = 0, want_V: bool = False, want_L: bool = False) -> dict:
    """Restarted GMRES driver (SURVEY §8(c) "Driver").  variant in
    {'mgs','igs1','igs2_two','igs2'} ('igs2' = Algorithm 3, one reduction)."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    n = A.n_rows
    rp, ci, vals = _csr64(A)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m1 = restart if 0 < restart < k else k
    x = np.empty(n)
    H = np.zeros((m1 + 1) * m1)
    res = np.full(k + 1, np.nan)
    V = np.zeros(n * (m1 + 1)) if want_V else None
    L = np.zeros(m1 * m1) if want_L else None
    ledger = np.zeros(k, dtype=np.int64)
    info = np.zeros(8, dtype=np.int64)
    trr = np.zeros(1)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    st = lib().oracle_gmres(n, _p(rp), _p(ci), _p(vals), _p(b), _p(x0a), int(k), int(restart),
                            float(tol), v, int(dot_block), _p(x), _p(H), _p(res), _p(V), _p(L),
                            _p(ledger), _p(info), _p(trr))
    if st != 0:
        raise ValueError(f"oracle_gmres status {st}")
    iters = int(info[0])
    out = dict(x=x, H=H.reshape(m1, m1 + 1).T, res_hist=res[:iters + 1], iters=iters,
               cycles=int(info[1]), term=TERM[int(info[2])], h_cols=int(info[3]),
               basis_cols=int(info[4]), priming_reductions=int(info[5]),
               ledger=ledger[:iters], true_relres=float(trr[0]), m=m1)
    if want_V:
        out["V"] = V.reshape(m1 + 1, n).T
    if want_L:
        out["L"] = L.reshape(m1, m1).T
    return out


def igs_qr(A, sweeps: int = 2, dot_block: int = 0):
    """Algorithm 1: Q, R, L with A = QR.  sweeps=1: one Gauss-Seidel iteration."""
    A = np.asfortranarray(A, dtype=np.float64)
    n, m = A.shape
    Q = np.zeros((n, m), order="F")
    R = np.zeros((m, m), order="F")
    L = np.zeros((m, m), order="F")
    ledger = np.zeros(m, dtype=np.int64)
    st = lib().oracle_igs_qr(n, m, _p(A), n, int(sweeps), int(dot_block), _p(Q), n, _p(R), _p(L), _p(ledger))
    if st != 0:
        raise ValueError(f"oracle_igs_qr status {st}")
    return Q, R, L, ledger


# ------------------------------------------------------------------ diagnostics
def norm2_estimate(A, rtol: float = 1e-4, maxit: int = 500) -> float:
    """||A||_2 by power iteration on A^T A from the normalised all-ones vector
    (reading R11)."""
    S = A.to_scipy()
    n = S.shape[1]
    x = np.ones(n) / np.sqrt(n)
    sigma = 0.0
    for _ in range(maxit):
        y = S.T @ (S @ x)
        ny = np.linalg.norm(y)
        if ny == 0.0:
            return 0.0
        new = np.sqrt(ny)
        x = y / ny
        if sigma > 0 and abs(new - sigma) <= rtol * new:
            return float(new)
        sigma = new
    return float(sigma)


def backward_error(A, b, x, normA: float) -> float:
    """beta(x) = ||b - A x|| / (||b|| + ||A||_2 ||x||)."""
    r = b - spmv(A, x)
    return float(np.linalg.norm(r) / (np.linalg.norm(b) + normA * np.linalg.norm(x)))


def loss_of_orthogonality(V, row_block: int = 0) -> float:
    """||I - V^T V||_F.  row_block > 0: V^T V summed over blocks of that many rows
    (the same sum over rows, in blocks, so a 100-column basis of 134M rows -- c5, 108 GB --
    needs no second copy of V), the block Grams added pairwise."""
    V = np.asarray(V)
    if row_block > 0:
        # block Grams added pairwise (a binary tree over the blocks, the same sum over rows):
        # the Gram of a 134M-row basis then carries O(log(blocks) eps) of rounding instead of
        # O(blocks eps), below the orthogonality it is there to measure
        stack = []
        for i in range(0, V.shape[0], row_block):
            B = np.array(V[i:i + row_block])
            G, lvl = B.T @ B, 0
            while stack and stack[-1][0] == lvl:
                G = stack.pop()[1] + G
                lvl += 1
            stack.append((lvl, G))
        G = stack.pop()[1]
        while stack:
            G = stack.pop()[1] + G
    else:
        G = V.T @ V
    return float(np.linalg.norm(np.eye(V.shape[1]) - G, "fro"))


def arnoldi_relation(A, V, H, p: int) -> float:
    """||A V_p - V_{p+1} H_{p+1,p}||_F / ||A||_F."""
    S = A.to_scipy()
    AV = S @ V[:, :p]
    F = AV - V[:, :p + 1] @ H[:p + 1, :p]
    return float(np.linalg.norm(F, "fro") / np.linalg.norm(S.data))


def kappa_Bk(A, b, V, p: int, x0=None) -> float:
    """kappa(B_k), B_k = [r0, A V_k]."""
    S = A.to_scipy()
    r0 = b - (S @ x0 if x0 is not None else 0.0)
    B = np.column_stack([r0, S @ V[:, :p]])
    s = np.linalg.svd(B, compute_uv=False)
    return float(s[0] / s[-1])


def S_norm(V, p: int) -> float:
    """||S_p||_2, S = (I + L^T)^{-1} L^T, L = strictly lower part of V_p^T V_p."""
    G = V[:, :p].T @ V[:, :p]
    Lt = np.triu(G, 1)
    S = np.linalg.solve(np.eye(p) + Lt, Lt)
    return float(np.linalg.norm(S, 2))


def sigma_min(V, p: int) -> float:
    """Smallest singular value of V_p (the plain definition, LAPACK SVD)."""
    return float(np.linalg.svd(np.asarray(V)[:, :p], compute_uv=False)[-1])


def column_normwise_diff(H1, H2, ncols: int) -> float:
    """max_j max_i |H1_ij - H2_ij| / max_i |H2_ij| over the first ncols columns
    (the parity metric of reading R9)."""
    worst = 0.0
    for j in range(ncols):
        ref = np.max(np.abs(H2[:j + 2, j]))
        d = np.max(np.abs(H1[:j + 2, j] - H2[:j + 2, j]))
        worst = max(worst, d / ref if ref > 0 else d)
    return float(worst)
