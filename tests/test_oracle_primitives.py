"""Pins for the oracle's primitives (CPU only).  Each pin is fixed by mathematics or by
a SPEC.md worked example (tests/golden/paper_values.json), never by the oracle itself."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
EPS = np.finfo(float).eps


def test_forward_solve_spec_example():
    ex = GOLD["spec_examples"]["forward_solve_unit"]
    L = np.zeros((2, 2)); L[1, 0] = ex["L21"]
    np.testing.assert_array_equal(oracle.forward_solve_unit(L, np.array(ex["b"])), ex["x"])


def test_forward_solve_ignores_upper_and_diagonal():
    rng = np.random.default_rng(5)
    L = np.tril(rng.uniform(-1, 1, (6, 6)), -1)
    b = rng.standard_normal(6)
    junk = L + np.triu(rng.uniform(-9, 9, (6, 6)))  # diag/upper must be ignored (unit lower)
    np.testing.assert_array_equal(oracle.forward_solve_unit(junk, b), oracle.forward_solve_unit(L, b))


@pytest.mark.parametrize("order", [1, 8, 50, 200])
def test_forward_solve_residual_bound(order):
    # Higham (cited at P:496-503): forward substitution is backward stable, so
    # |(I+L)x - b| <= gamma_order |I+L| |x| componentwise; checked with the dense product
    rng = np.random.default_rng(order)
    L = np.tril(rng.uniform(-1, 1, (order, order)), -1)
    b = rng.standard_normal(order)
    x = oracle.forward_solve_unit(L, b)
    M = np.eye(order) + L
    r = M @ x - b
    gam = order * EPS / (1 - order * EPS)
    assert np.all(np.abs(r) <= 2 * gam * (np.abs(M) @ np.abs(x)) + 1e-300)
    # S:106 normwise form for the small-L regime the algorithm lives in (||L|| ~ eps kappa)
    Ls = L * 1e-3
    xs_ = oracle.forward_solve_unit(Ls, b)
    rs = (np.eye(order) + Ls) @ xs_ - b
    assert np.linalg.norm(rs) <= 100 * order * EPS * np.linalg.norm(b) * (1 + np.linalg.norm(Ls))
    # and against LAPACK's triangular solve
    import scipy.linalg as sl
    ref = sl.solve_triangular(np.eye(order) + Ls, b, lower=True, unit_diagonal=True)
    assert np.allclose(xs_, ref, rtol=1e-13, atol=1e-14 * np.abs(ref).max())


def test_hessenberg_lsq_spec_examples():
    for key in ("hessenberg_lsq_exact", "hessenberg_lsq_ls"):
        ex = GOLD["spec_examples"][key]
        y, res = oracle.hessenberg_lsq(np.array(ex["H"]), ex["rho"])
        np.testing.assert_allclose(y, ex["y"], rtol=0, atol=1e-15)
        assert abs(res - ex["residual"]) <= 1e-15


@pytest.mark.parametrize("p", [1, 5, 10, 40])
def test_hessenberg_lsq_vs_dense_lstsq(p):
    # random (p+1) x p upper Hessenberg vs a dense least-squares solve
    rng = np.random.default_rng(p)
    H = np.triu(rng.standard_normal((p + 1, p)), -1)
    rho = 2.5
    y, res = oracle.hessenberg_lsq(H, rho)
    e1 = np.zeros(p + 1); e1[0] = rho
    ys, *_ = np.linalg.lstsq(H, e1, rcond=None)
    assert np.allclose(y, ys, rtol=1e-10, atol=1e-12)
    assert abs(res - np.linalg.norm(e1 - H @ ys)) <= 1e-12 * rho


def test_dot_and_norm_examples():
    for v, nrm in GOLD["spec_examples"]["norm2"]["cases"]:
        v = np.array(v)
        assert np.sqrt(oracle.dot(v, v)) == nrm
    ex = GOLD["spec_examples"]["block_inner"]
    Q = np.eye(3)[:, :2]
    x = np.array(ex["x"])
    out = oracle.block_dot(Q, x, np.zeros(3))
    np.testing.assert_array_equal(out[:2], ex["result"])
    assert out[2] == x @ x and out[5] == 0.0


@pytest.mark.parametrize("block", [0, 7, 64, 1000])
def test_dot_reduction_orders_agree(block):
    rng = np.random.default_rng(11)
    a, b = rng.standard_normal(5001), rng.standard_normal(5001)
    exact = float(np.dot(a.astype(np.longdouble), b.astype(np.longdouble)))
    bound = 5001 * EPS * np.dot(np.abs(a), np.abs(b))      # Higham's gamma_n bound
    assert abs(oracle.dot(a, b, block) - exact) <= bound


def test_dot_blocked_is_exactly_the_stated_order():
    # blocked knob == sequential sum of sequential block sums, written out here in Python
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(103), rng.standard_normal(103)
    parts = []
    for i0 in range(0, 103, 10):
        s = 0.0
        for i in range(i0, min(i0 + 10, 103)):
            s += a[i] * b[i]
        parts.append(s)
    tot = 0.0
    for s in parts:
        tot += s
    assert oracle.dot(a, b, 10) == tot


def test_spmv_walker_example_and_dense():
    ex = GOLD["spec_examples"]["matvec_walker4"]
    A, _ = W.walker(ex["n"], ex["alpha"])
    e4 = np.zeros(4); e4[3] = 1.0
    np.testing.assert_array_equal(oracle.spmv(A, e4), ex["y"])
    P = W.config("c3", N=12)
    x = np.random.default_rng(1).standard_normal(P.A.n_cols)
    D = P.A.to_dense()
    assert np.allclose(oracle.spmv(P.A, x), D @ x, rtol=0, atol=10 * EPS * np.abs(D).sum(1).max() * np.abs(x).max())


def test_block_dot_layout_matches_definition():
    rng = np.random.default_rng(2)
    V = rng.standard_normal((300, 7)); u = rng.standard_normal(300); z = rng.standard_normal(300)
    out = oracle.block_dot(V, u, z)
    M = np.column_stack([V, u]).T @ np.column_stack([u, z])    # [V, u]^T [u, z]
    ref = np.concatenate([M[:7, 0], [M[7, 0]], M[:7, 1], [M[7, 1]]])
    assert np.allclose(out, ref, rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------- Algorithm 1 (QR)
def test_igs_qr_identity():
    Q, R, L, _ = oracle.igs_qr(np.eye(12)[:, :7])
    np.testing.assert_allclose(Q, np.eye(12)[:, :7], atol=1e-16)
    np.testing.assert_allclose(R, np.eye(7), atol=1e-16)


@pytest.mark.parametrize("sweeps", [1, 2])
def test_igs_qr_vs_householder(sweeps):
    rng = np.random.default_rng(4)
    A = rng.standard_normal((50, 20))
    Q, R, L, led = oracle.igs_qr(A, sweeps)
    Qh, Rh = np.linalg.qr(A)                     # LAPACK Householder QR, signs normalised
    Rh = np.sign(np.diag(Rh))[:, None] * Rh
    assert np.abs(R - Rh).max() <= 1e-12 * np.abs(Rh).max()
    assert np.allclose(np.triu(R), R)            # upper triangular, positive diagonal
    assert np.all(np.diag(R) > 0)
    assert np.linalg.norm(A - Q @ R) <= 1e-14 * np.linalg.norm(A)
    assert np.linalg.norm(np.eye(20) - Q.T @ Q) <= 1e-14
    assert list(led[:2]) == [1, 1] and np.all(led[2:] == sweeps)   # 'Global Synchronization' count


def _graded(n=60, m=30, kappa=1e10, seed=5):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    Wm, _ = np.linalg.qr(rng.standard_normal((m, m)))
    return (U * np.logspace(0, -np.log10(kappa), m)) @ Wm.T


def test_igs_qr_two_sweeps_eps_orthogonality_graded():
    # with two Gauss-Seidel iterations the loss of orthogonality is O(eps) even for
    # kappa(A) = 1e10; one iteration only O(eps) kappa(A)
    A = _graded()
    kappa = np.linalg.cond(A)
    Q2, R2, _, _ = oracle.igs_qr(A, 2)
    Q1, R1, _, _ = oracle.igs_qr(A, 1)
    loo2 = np.linalg.norm(np.eye(30) - Q2.T @ Q2)
    loo1 = np.linalg.norm(np.eye(30) - Q1.T @ Q1)
    assert loo2 <= 1e-13
    assert loo1 <= 10 * EPS * kappa and loo1 >= 1e3 * loo2
    for Q, R in ((Q1, R1), (Q2, R2)):            # both are backward stable factorizations
        assert np.linalg.norm(A - Q @ R) <= 1e-14 * np.linalg.norm(A)


def test_igs_qr_step7_reading():
    # reading R22: only the entry of r^(0) belonging to the lagged-normalised q_{k-1} is divided
    # by gamma_{k-1}; dividing the whole column (the literal print) breaks A = QR
    A = np.random.default_rng(6).standard_normal((40, 10))
    Q, R, _, _ = oracle.igs_qr(A)
    R_lit = R.copy()
    for k in range(2, 10):
        R_lit[:k - 1, k] /= R[k - 1, k - 1]
    assert np.linalg.norm(A - Q @ R) <= 1e-14 * np.linalg.norm(A)
    assert np.linalg.norm(A - Q @ R_lit) >= 1e-2 * np.linalg.norm(A)


# ------------------------------------------------------------- basis diagnostics
def test_S_norm_closed_forms():
    # orthonormal basis: S = 0; two columns at angle theta: U = [[0, cos]], S = U, ||S|| = |cos|;
    # a repeated column (orthogonality lost): ||S||_2 = 1 exactly (Paige)
    rng = np.random.default_rng(8)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 6)))
    assert oracle.S_norm(Q, 6) <= 1e-15
    th = 0.3
    V = np.zeros((5, 2)); V[0, 0] = 1.0; V[0, 1] = np.cos(th); V[1, 1] = np.sin(th)
    assert abs(oracle.S_norm(V, 2) - np.cos(th)) <= 1e-15
    W = np.column_stack([Q[:, 0], Q[:, 1], Q[:, 0]])
    assert abs(oracle.S_norm(W, 3) - 1.0) <= 1e-14


def test_sigma_min_known_spectrum():
    rng = np.random.default_rng(9)
    U, _ = np.linalg.qr(rng.standard_normal((50, 7)))
    Wm, _ = np.linalg.qr(rng.standard_normal((7, 7)))
    s = np.array([3.0, 2.0, 1.0, 0.5, 0.1, 1e-3, 2.5])
    V = (U * s) @ Wm.T
    assert abs(oracle.sigma_min(V, 7) - 1e-3) <= 1e-14
    assert abs(oracle.sigma_min(U, 7) - 1.0) <= 1e-14


def test_backward_error_spec_example_x0():
    """beta(0) = ||b|| / (||b|| + ||A|| * 0) = 1, whatever A, b and ||A||."""
    ex = GOLD["spec_examples"]["backward_error_x0"]
    A = W.config("c1").A
    b = np.random.default_rng(3).standard_normal(A.n_rows)
    for normA in (1.0, 3.7, 1e6):
        assert oracle.backward_error(A, b, np.zeros(A.n_rows), normA) == ex["beta"]


def test_backward_error_exact_solution_and_scaling():
    """beta(x) = 0 for the exact solution of a system the oracle SpMV reproduces exactly
    (integer data), and beta is invariant under b, x -> s b, s x (homogeneous of degree 0)."""
    A = W.tridiag_csr(50, -1.0, 4.0, -2.0)
    x = np.arange(1.0, 51.0)
    b = oracle.spmv(A, x)
    assert oracle.backward_error(A, b, x, 6.0) == 0.0
    rng = np.random.default_rng(9)
    xa = x + 1e-3 * rng.standard_normal(50)
    b1 = oracle.backward_error(A, b, xa, 6.0)
    b2 = oracle.backward_error(A, 8.0 * b, 8.0 * xa, 6.0)   # powers of 2: exact scaling
    assert b1 > 0 and b1 == b2
    # against the definition written out with a dense matrix (independent of oracle.spmv)
    D = A.to_dense()
    ref = np.linalg.norm(b - D @ xa) / (np.linalg.norm(b) + 6.0 * np.linalg.norm(xa))
    assert abs(b1 - ref) <= 1e-12 * ref


def test_column_normwise_diff_detects_differences():
    """The parity metric every GPU test rests on (reading R9): zero for identical H, exactly
    the perturbation relative to the column's max for one changed entry, blind to columns past
    ncols, and it sees a sign flip, a transposed pair and a shifted column."""
    rng = np.random.default_rng(4)
    m = 12
    H = np.triu(rng.standard_normal((m + 1, m)), -1)
    assert oracle.column_normwise_diff(H, H.copy(), m) == 0.0
    G = H.copy()
    G[3, 5] += 1e-9
    want = 1e-9 / np.max(np.abs(H[:7, 5]))
    assert abs(oracle.column_normwise_diff(G, H, m) - want) <= 1e-6 * want
    assert oracle.column_normwise_diff(G, H, 5) == 0.0        # column 5 not compared
    S = H.copy(); S[2, 4] = -S[2, 4]                          # a dropped sign
    assert oracle.column_normwise_diff(S, H, m) >= 2 * abs(H[2, 4]) / np.max(np.abs(H[:6, 4])) * (1 - 1e-12)
    T = H.copy(); T[[1, 2], 6] = T[[2, 1], 6]                 # two entries swapped
    assert oracle.column_normwise_diff(T, H, m) > 1e-3
    Z = H.copy(); Z[:, 7] = np.roll(H[:, 7], 1)               # off by one row
    assert oracle.column_normwise_diff(Z, H, m) > 1e-3
    # entries below the subdiagonal are outside the metric (the Hessenberg structure)
    B = H.copy(); B[10, 2] = 1.0
    assert oracle.column_normwise_diff(B, H, m) == 0.0


def test_loss_of_orthogonality_closed_forms_and_row_blocks():
    """||I - V^T V||_F against closed forms -- an orthonormal Q (QR) gives O(eps),
    V = [e1, e1] gives ||[[0,-1],[-1,0]]||_F = sqrt(2), V = 2 I_k gives 3 sqrt(k) -- and the
    row-blocked Gram (used for the 108 GB c5 basis) agrees with the one-shot Gram, including a
    ragged last block."""
    rng = np.random.default_rng(11)
    Q, _ = np.linalg.qr(rng.standard_normal((1000, 20)))
    assert oracle.loss_of_orthogonality(Q) <= 1e-14
    E = np.zeros((50, 2)); E[0, :] = 1.0
    assert abs(oracle.loss_of_orthogonality(E) - np.sqrt(2.0)) <= 1e-15
    assert abs(oracle.loss_of_orthogonality(2.0 * np.eye(7)) - 3.0 * np.sqrt(7.0)) <= 1e-14
    V = np.asfortranarray(rng.standard_normal((1003, 9)) * 0.3)
    full = oracle.loss_of_orthogonality(V)
    for rb in (1, 7, 1000, 5000):
        assert abs(oracle.loss_of_orthogonality(V, row_block=rb) - full) <= 1e-13 * full
    assert abs(oracle.loss_of_orthogonality(Q, row_block=64) - oracle.loss_of_orthogonality(Q)) <= 1e-14
    # the blocked form is accurate where a long running sum is not: one normalised constant
    # column of 3 * 2^20 rows has ||I - V^T V||_F = 0 up to rounding (a running sum of its
    # 3M squares drifts by ~1e-10)
    n = 3 << 20
    c = np.full((n, 1), 1.0 / np.sqrt(n))
    assert oracle.loss_of_orthogonality(c, row_block=4096) <= 1e-13


def test_dot_pairwise_block_mode():
    """oracle.dot with block = -B (blocks of B, block sums added pairwise; reading R27):
    exact where every order is exact, the same value as the running-sum modes up to rounding,
    and accurate where a running sum over many blocks is not: a normalised constant vector of
    3 * 2^20 entries has v.v = 1 up to rounding."""
    x = np.ldexp(np.arange(1, 100001, dtype=np.float64), -20)   # products and sums exact
    exact = float(np.sum(x * x))
    assert oracle.dot(x, x, -512) == oracle.dot(x, x, 512) == oracle.dot(x, x, 0) == exact
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal(70001), rng.standard_normal(70001)
    ref = float(np.dot(a, b))
    for blk in (-1, -7, -4096, -70001, -100000):
        assert abs(oracle.dot(a, b, blk) - ref) <= 1e-12 * np.abs(a) @ np.abs(b)
    n = 3 << 20
    v = np.full(n, 1.0 / np.sqrt(n))
    assert abs(oracle.dot(v, v, -4096) - 1.0) <= 1e-13
    assert abs(oracle.dot(v, v, 0) - 1.0) >= 1e-12   # (the single running sum: ~5e-11)

