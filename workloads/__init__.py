"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no Arnoldi, no Gram-Schmidt, no
least squares).  It only builds matrices in CSR form and right-hand sides, from
the recipes in DESIGN.md §"Input recipe" (= SURVEY.md §8(d), BASELINE.json
`configs`).  Random numbers come from numpy `default_rng(seed)` (PCG64) only.

Every stencil entry is produced by the same IEEE expression sequence
    h = 1.0 / (N + 1);  lo = -1.0 - (beta * h) / 2.0;  hi = -1.0 + (beta * h) / 2.0
so a shard generated for rows [r0, r1) is bitwise identical to the same rows of
the whole matrix.

CSR convention used everywhere in this repo:
    rowptr : int64[n_rows + 1], local offsets (rowptr[0] == 0)
    colind : int32 or int64, GLOBAL column indices, strictly increasing per row
    values : float64
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Csr", "Problem", "stencil_csr", "tridiag_csr", "dense_upper_csr", "dense_to_csr",
    "config", "CONFIGS", "matvec_ones_host",
    "simoncini", "walker", "embree", "helmert", "diag_csr",
]


@dataclasses.dataclass
class Csr:
    n_rows: int            # rows in this block
    n_cols: int            # global columns
    row_begin: int         # global index of the first row of this block
    rowptr: np.ndarray     # int64 [n_rows+1]
    colind: np.ndarray     # int32/int64 [nnz]
    values: np.ndarray     # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    @property
    def index_bits(self) -> int:
        return 64 if self.colind.dtype == np.int64 else 32

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.colind.astype(np.int64), self.rowptr),
                             shape=(self.n_rows, self.n_cols))

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()


@dataclasses.dataclass
class Problem:
    name: str
    A: Csr
    b: np.ndarray                 # float64 [n]
    k: int                        # max Arnoldi iterations
    restart: int                  # 0 => unrestarted
    tol: float                    # 0 => run exactly k
    note: str = ""


# --------------------------------------------------------------------------------------
# convection-diffusion stencils (c1, c3, c4, c5)
# --------------------------------------------------------------------------------------

def _stencil_coeffs(N: int, betas):
    h = 1.0 / (N + 1)
    lo = [-1.0 - (float(bt) * h) / 2.0 for bt in betas]   # west / south / down
    hi = [-1.0 + (float(bt) * h) / 2.0 for bt in betas]   # east / north / up
    return lo, hi


def stencil_csr(N: int, dim: int, betas, row_begin: int = 0, row_end: int | None = None,
                index_bits: int = 32) -> Csr:
    """h^2-scaled centred convection-diffusion on an N^dim interior grid, Dirichlet,
    x-fastest ordering (row = i + N*j + N*N*l).  Diagonal 2*dim, neighbour in
    direction d at offset -N^d gets lo[d] = -1 - beta_d h/2, at +N^d gets hi[d].
    Rows [row_begin, row_end) only, columns global."""
    n = N ** dim
    if row_end is None:
        row_end = n
    assert 0 <= row_begin <= row_end <= n
    lo, hi = _stencil_coeffs(N, betas)
    rows = np.arange(row_begin, row_end, dtype=np.int64)
    m = rows.size
    coord = []
    r = rows.copy()
    for _ in range(dim):
        coord.append(r % N)
        r //= N
    # neighbour slots in increasing column order: -N^(dim-1) ... -1, 0, +1 ... +N^(dim-1)
    offs, vals, valid = [], [], []
    for d in reversed(range(dim)):
        offs.append(-(N ** d)); vals.append(lo[d]); valid.append(coord[d] > 0)
    offs.append(0); vals.append(float(2 * dim)); valid.append(np.ones(m, dtype=bool))
    for d in range(dim):
        offs.append(N ** d); vals.append(hi[d]); valid.append(coord[d] < N - 1)
    S = len(offs)
    mask = np.stack(valid, axis=1)                       # [m, S]
    counts = mask.sum(axis=1)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    idt = np.int64 if index_bits == 64 else np.int32
    cols = (rows[:, None] + np.asarray(offs, dtype=np.int64)[None, :])[mask].astype(idt)
    v = np.broadcast_to(np.asarray(vals, dtype=np.float64)[None, :], (m, S))[mask].copy()
    return Csr(m, n, row_begin, rowptr, cols, v)


def tridiag_csr(n: int, sub: float, diag: float, sup: float) -> Csr:
    """Config c1 operator: tridiag(sub, diag, super), taken literally from BASELINE.json
    configs[0] ("diag 2+0.5, sub -1-0.5, super -1+0.5")."""
    rows = np.arange(n, dtype=np.int64)
    offs = np.array([-1, 0, 1])
    vals = np.array([sub, diag, sup], dtype=np.float64)
    mask = np.stack([rows > 0, np.ones(n, bool), rows < n - 1], axis=1)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rowptr[1:])
    cols = (rows[:, None] + offs[None, :])[mask].astype(np.int32)
    v = np.broadcast_to(vals[None, :], (n, 3))[mask].copy()
    return Csr(n, n, 0, rowptr, cols, v)


def dense_to_csr(D: np.ndarray, keep_zeros_upper: bool = False) -> Csr:
    """Dense -> CSR dropping exact zeros (or keeping the whole upper triangle)."""
    n_rows, n_cols = D.shape
    if keep_zeros_upper:
        mask = np.triu(np.ones_like(D, dtype=bool))
    else:
        mask = D != 0.0
    counts = mask.sum(axis=1)
    rowptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    cols = np.nonzero(mask)[1].astype(np.int32)
    vals = D[mask].astype(np.float64)
    return Csr(n_rows, n_cols, 0, rowptr, cols, vals)


def dense_upper_csr(n: int = 2000, seed: int = 1) -> Csr:
    """Config c2: A = diag(linspace(1,1000,n)) + triu(G,1)*2/sqrt(n), G ~ N(0,1) from
    default_rng(seed); stored as CSR of the full upper triangle incl. the diagonal."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n))
    A = np.triu(G, 1) * (2.0 / math.sqrt(n))
    A[np.diag_indices(n)] = np.linspace(1.0, 1000.0, n)
    return dense_to_csr(A, keep_zeros_upper=True)


def diag_csr(d) -> Csr:
    d = np.asarray(d, dtype=np.float64)
    n = d.size
    return Csr(n, n, 0, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), d.copy())


def matvec_ones_host(A: Csr) -> np.ndarray:
    """b = A*ones as per-row sums of the CSR values (input recipe "b = A*ones",
    BASELINE.json configs 2,3,5).  Input preparation, not part of the method: both the
    oracle and the CUDA path receive the same b bytes."""
    out = np.empty(A.n_rows, dtype=np.float64)
    # np.add.reduceat sums each segment sequentially left to right
    nonempty = A.rowptr[1:] > A.rowptr[:-1]
    out[:] = 0.0
    if A.nnz:
        sums = np.add.reduceat(A.values, A.rowptr[:-1][nonempty])
        out[nonempty] = sums
    return out


# --------------------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------------------

C3_BETA = (50.0, 50.0)
C4_BETA = (100.0, 50.0, 25.0)
C5_BETA = (20.0, 20.0, 20.0)


def config(name: str, *, N: int | None = None, row_begin: int = 0, row_end: int | None = None,
           k: int | None = None) -> Problem:
    """Build config `name` in {c1..c5}. `N` overrides the grid size for the stencils
    (downsized parity cases); `row_begin/row_end` build one row block (shard)."""
    if name == "c1":
        n = 1000
        A = tridiag_csr(n, sub=-1.0 - 0.5, diag=2.0 + 0.5, sup=-1.0 + 0.5)
        b = np.random.default_rng(0).uniform(-1.0, 1.0, n)
        return Problem("c1", A, b, k or 60, 0, 0.0, "1D tridiagonal, b~U(-1,1) seed 0")
    if name == "c2":
        A = dense_upper_csr(2000, 1)
        b = matvec_ones_host(A)
        return Problem("c2", A, b, k or 300, 0, 0.0, "dense non-normal upper triangular, b=A*1")
    if name == "c3":
        N = N or 1024
        A = stencil_csr(N, 2, C3_BETA, row_begin, row_end)
        b = matvec_ones_host(A)
        return Problem("c3", A, b, k or 300, 0, 0.0, f"2D 5-point {N}^2, b=A*1")
    if name == "c4":
        N = N or 256
        A = stencil_csr(N, 3, C4_BETA, row_begin, row_end)
        b_full = np.random.default_rng(3).uniform(0.0, 1.0, N ** 3)
        b = b_full[A.row_begin:A.row_begin + A.n_rows].copy()
        return Problem("c4", A, b, k or 2000, 100, 1e-12, f"3D 7-point {N}^3 GMRES(100), b~U(0,1) seed 3")
    if name == "c5":
        N = N or 512
        A = stencil_csr(N, 3, C5_BETA, row_begin, row_end, index_bits=64)
        b = matvec_ones_host(A)
        return Problem("c5", A, b, k or 100, 0, 0.0, f"3D 7-point {N}^3 int64, b=A*1")
    raise KeyError(name)


CONFIGS = ("c1", "c2", "c3", "c4", "c5")


# --------------------------------------------------------------------------------------
# generator-defined matrices from the paper's §5 (oracle pins only)
# --------------------------------------------------------------------------------------

def simoncini(n: int = 100, seed: int = 0):
    """A = diag(1e-4, 2, 3, ..., n) (§5 "Ill-Conditioned Diagonal Matrix",
    P:1269-1272); b = randn(n) normalised to ||b||=1 (seed is ours)."""
    d = np.arange(1, n + 1, dtype=np.float64)
    d[0] = 1e-4
    b = np.random.default_rng(seed).standard_normal(n)
    b /= np.linalg.norm(b)
    return diag_csr(d), b


def walker(n: int = 10, alpha: float = 2000.0):
    """Walker's matrix, PAPER.md eq. (walker): diag(1..n) with A[0,n-1]=alpha,
    b = ones."""
    D = np.diag(np.arange(1, n + 1, dtype=np.float64))
    D[0, n - 1] = alpha
    return dense_to_csr(D), np.ones(n)


def embree(n: int = 100, delta: float = 0.1):
    """Embree's delta-bidiagonal: ones on the diagonal, delta on the
    superdiagonal (reading R18: n=100, delta=0.1, b=ones)."""
    D = np.eye(n) + delta * np.eye(n, k=1)
    return dense_to_csr(D), np.ones(n)


def helmert(n: int = 18):
    """Helmert matrix (orthogonal): first row ones/sqrt(n); row i>=1 has
    ones in columns < i and -i at column i, scaled by 1/sqrt(i(i+1))."""
    Q = np.zeros((n, n))
    Q[0, :] = 1.0 / math.sqrt(n)
    for i in range(1, n):
        Q[i, :i] = 1.0
        Q[i, i] = -float(i)
        Q[i, :] /= math.sqrt(i * (i + 1.0))
    return dense_to_csr(Q), np.ones(n)
