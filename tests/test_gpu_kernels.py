"""Per-kernel parity: each libigs kernel (through the C ABI) against the oracle's
primitive on the same seeded inputs, at sizes spanning several tiles plus a ragged tail."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2205_07805_b200 as P
    P.lib()
    return torch


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [5, 1024 * 3 + 17, 70001, 1 << 20, 2 * 740 * 512 + 777])
@pytest.mark.parametrize("p", [0, 1, 7, 64, 300])
def test_block_dot_vs_oracle(torch_cuda, n, p):
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    if n == 1 << 20 and p == 300:
        p = 100
    # (n = 2 * 740 * 512 + 777: three rounds of the column-sweep kernel -- 148 CTAs x 5 tiles --
    #  the last with two tiles, one of them partial; p >= 96 takes that kernel)
    rng = np.random.default_rng(n + p)
    ld = n + (n % 2) + 32           # padded, even
    Vh = rng.standard_normal((p + 1, ld))   # column-major storage: row j = column j
    Vh[:, n:] = np.nan                      # padding must never be read as data
    u = Vh[p, :n].copy(); z = rng.standard_normal(n)
    Vd = _dev(torch, Vh.reshape(-1))
    ud = Vd[p * ld: p * ld + n]             # u = V[:, p] as in the solver
    zd = _dev(torch, z)
    for nv in (1, 2):
        out = torch.empty(2 * (p + 1), dtype=torch.float64, device="cuda")
        P.igs_op_block_dot(n, p, Vd, ld, ud, zd if nv == 2 else None, out)
        got = out.cpu().numpy()
        Vp = Vh[:p, :n].T
        ref = oracle.block_dot(Vp, u, z, block=4096)
        scale = np.concatenate([np.abs(Vp).T @ np.abs(u), [np.abs(u) @ np.abs(u)],
                                np.abs(Vp).T @ np.abs(z), [np.abs(u) @ np.abs(z)]])
        m = (p + 1) if nv == 1 else 2 * (p + 1)
        err = np.abs(got[:m] - ref[:m]) / scale[:m]
        assert np.all(err <= 64 * EPS * np.log2(n + 2)), (nv, err.max())


def test_block_dot_deterministic(torch_cuda):
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    n, p = 300001, 50
    rng = np.random.default_rng(7)
    V = _dev(torch, rng.standard_normal((p + 1) * (n + 1)))
    z = _dev(torch, rng.standard_normal(n + 1))
    outs = []
    for _ in range(3):
        o = torch.empty(2 * (p + 1), dtype=torch.float64, device="cuda")
        P.igs_op_block_dot(n, p, V, n + 1, V[p * (n + 1):], z, o)
        outs.append(o.cpu().numpy().tobytes())
    assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("n", [1, 2, 511, 1 << 16 | 3])
@pytest.mark.parametrize("p", [0, 1, 9, 64, 300])
@pytest.mark.parametrize("gs", [1, 2])
def test_update_vs_oracle(torch_cuda, n, p, gs):
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    rng = np.random.default_rng(3 * n + p)
    ld = n + (n % 2)
    Vh = np.zeros((p + 2, ld)); Vh[:, :n] = rng.standard_normal((p + 2, n))
    z = rng.standard_normal(n)
    alpha = rng.standard_normal(p) * 1e-3 if gs == 2 else None
    beta = rng.standard_normal(p + 1)
    gamma = 0.75
    Vp = Vh[:p, :n].T
    u = Vh[p, :n].copy()
    v_ref, un_ref = oracle.update(Vp, u, z, alpha, beta, gamma)
    Vd = _dev(torch, Vh.reshape(-1))
    zd = _dev(torch, np.concatenate([z, [0.0] * (ld - n)]))
    ad = _dev(torch, alpha) if alpha is not None else None
    bd = _dev(torch, beta)
    P.igs_op_update(n, p, Vd, ld, Vd[p * ld:], zd, ad, bd, gamma, Vd[p * ld:], Vd[(p + 1) * ld:])
    out = Vd.cpu().numpy().reshape(p + 2, ld)
    scale_v = (np.abs(u) + (np.abs(Vp) @ np.abs(alpha) if alpha is not None else 0)) / gamma
    assert np.all(np.abs(out[p, :n] - v_ref) <= 8 * (p + 2) * EPS * scale_v + 1e-300)
    scale_u = np.abs(z) / gamma + np.abs(np.column_stack([Vp, v_ref])) @ np.abs(beta)
    assert np.all(np.abs(out[p + 1, :n] - un_ref) <= 8 * (p + 2) * EPS * scale_u + 1e-300)
    assert np.all(out[:p, :n] == Vh[:p, :n])           # V_p untouched


@pytest.mark.parametrize("order", [1, 7, 64, 300])
def test_trisolve_vs_oracle(torch_cuda, order):
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    rng = np.random.default_rng(order)
    L = np.tril(rng.uniform(-1, 1, (order, order)), -1) * 1e-2
    b = rng.standard_normal(order)
    ref = oracle.forward_solve_unit(L, b)
    Ld = _dev(torch, np.asfortranarray(L).reshape(-1, order="F"))
    xd = torch.empty(order, dtype=torch.float64, device="cuda")
    P.igs_op_trisolve(order, Ld, order, _dev(torch, b), xd)
    got = xd.cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-14, atol=1e-14 * np.abs(ref).max())


def _csr_random(n, rng):
    lens = rng.integers(0, 40, n)
    lens[::17] = 0
    lens[5::97] = 300          # a few long rows
    rows = []
    cols = []
    for i, L in enumerate(lens):
        L = min(L, n)
        c = np.sort(rng.choice(n, L, replace=False))
        cols.append(c)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([c.size for c in cols], out=rowptr[1:])
    colind = np.concatenate(cols).astype(np.int32)
    return W.Csr(n, n, 0, rowptr, colind, rng.standard_normal(colind.size))


@pytest.mark.parametrize("name", ["c1", "c2", "c3_64", "c4_24", "c5_12", "random"])
def test_spmv_vs_oracle(torch_cuda, name):
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    rng = np.random.default_rng(1)
    if name == "random":
        A = _csr_random(3001, rng)
    elif "_" in name:
        cfg, N = name.split("_")
        A = W.config(cfg, N=int(N)).A
    else:
        A = W.config(name).A
    s = P.Solver(A)
    x = rng.standard_normal(A.n_rows)
    y = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    s.spmv(_dev(torch, x), y)
    ref = oracle.spmv(A, x)
    absA = W.Csr(A.n_rows, A.n_cols, 0, A.rowptr, A.colind, np.abs(A.values))
    bound = 4 * EPS * np.diff(A.rowptr).clip(1) * oracle.spmv(absA, np.abs(x))
    assert np.all(np.abs(y.cpu().numpy() - ref) <= bound + 1e-300)
    s.close()


# ---------------------------------------- SELL-32 diagonal slices (a1 SpMV)
def _csr_banded(n, offs, drop, rng, scatter_rows=0, dtype=np.int32):
    """Rows r with columns r + o (o in offs, inside [0, n)), each entry dropped with
    probability `drop` (row masks vary inside a slice; some rows end up empty); the first
    `scatter_rows` rows get three more columns anywhere in the row (their slices then hold
    far more than 8 distinct offsets).  Columns strictly increasing per row (igs.h)."""
    cols = []
    for r in range(n):
        c = np.array([r + o for o in offs if 0 <= r + o < n and rng.random() >= drop], dtype=np.int64)
        if r < scatter_rows:
            c = np.union1d(c, rng.integers(0, n, 3))
        cols.append(c)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([c.size for c in cols], out=rowptr[1:])
    colind = np.concatenate(cols).astype(dtype)
    return W.Csr(n, n, 0, rowptr, colind, rng.standard_normal(colind.size))


def _sell_case(name):
    rng = np.random.default_rng(7)
    if name == "band7_masked":      # 7 offsets, 20% of entries missing, ragged last slice
        return _csr_banded(5013, [-70, -7, -1, 0, 1, 7, 70], 0.2, rng), "all"
    if name == "band9":             # 9 distinct offsets: explicit slices but at the two ends
        return _csr_banded(2000, [-90, -40, -9, -1, 0, 1, 9, 40, 90], 0.2, rng), "ends"
    if name == "band8_mixed":       # rows 0..99 with scattered columns: their slices explicit, the rest diagonal
        return _csr_banded(3001, [-300, -17, -1, 0, 1, 17, 300, 301], 0.1, rng, scatter_rows=100), "some"
    if name == "band5_int64":
        return _csr_banded(4099, [-64, -1, 0, 1, 64], 0.05, rng, dtype=np.int64), "all"
    A = W.config(name.split("_")[0], N=int(name.split("_")[1])).A if "_" in name else W.config(name).A
    return A, "most"


@pytest.mark.parametrize("diag", ["1", "0", "walk"])
@pytest.mark.parametrize("name", ["band7_masked", "band9", "band8_mixed", "band5_int64", "c1", "c4_24", "c4_33", "c5_12",
                                  "c3_600"])
def test_sell_diag_slices_bitwise(torch_cuda, name, diag, monkeypatch):
    """The SELL-32 copy with diagonal slices (column = row + the slice's offset picked by the
    row's mask) and with every slice explicit (IGS_SELL_DIAG=0) both equal the oracle's row
    loop (P:1059 Step 4) bit for bit; the slice classification is the one the matrix implies.
    "walk": all-diagonal matrices through the kernel of resident warps walking slices at any size
    (IGS_SELL_WALK_MIN_N=0; by default from 262144 rows on -- c3_600 takes it either way)."""
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    monkeypatch.setenv("IGS_SELL_DIAG", "0" if diag == "0" else "1")
    if diag == "walk":
        monkeypatch.setenv("IGS_SELL_WALK_MIN_N", "0")
    A, expect = _sell_case(name)
    s = P.Solver(A)
    info = s.info()
    assert info["sell"] == 1
    ns = (A.n_rows + 31) // 32
    nd = info["sell_diag_slices"]
    assert info["sell_walk"] == int(nd == ns and (diag == "walk" or A.n_rows >= 262144))
    if diag == "0":
        assert nd == 0
    elif expect == "ends":          # rows within 90 of either end miss an offset: <= 8 left
        assert 0 < nd <= 2 * (90 // 32 + 1)
    elif expect == "all":
        assert nd == ns
    else:
        assert 0 < nd < ns or (expect == "most" and nd == ns)
    rng = np.random.default_rng(11)
    for _ in range(2):
        x = rng.standard_normal(A.n_rows)
        y = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
        s.spmv(_dev(torch, x), y)
        assert y.cpu().numpy().tobytes() == oracle.spmv(A, x).tobytes()
    s.close()


@pytest.mark.parametrize("N", [24, 66])
def test_sell_diag_slices_solve_bitwise(torch_cuda, N, monkeypatch):
    """A GMRES(30) Alg. 3 cycle (persistent kernel at 24^3, graph-replayed kernels at 66^3,
    where the SpMV and the cycle-end residual take the slice-walking kernel) gives the
    same H, residual history and x bit for bit with diagonal slices, without them, and with
    diagonal slices but the one-thread-per-row kernel (IGS_SELL_WALK_MIN_N=-1)."""
    torch = torch_cuda
    import paper_2205_07805_b200 as P
    prob = W.config("c4", N=N)
    out = {}
    for diag, walk in (("1", None), ("0", None), ("1", "-1")):
        monkeypatch.setenv("IGS_SELL_DIAG", diag)
        if walk is None:
            monkeypatch.delenv("IGS_SELL_WALK_MIN_N", raising=False)
        else:
            monkeypatch.setenv("IGS_SELL_WALK_MIN_N", walk)
        s = P.Solver(prob.A)
        assert (s.info()["sell_diag_slices"] > 0) == (diag == "1")
        assert s.info()["sell_walk"] == int(diag == "1" and walk is None and N == 66)
        b = _dev(torch, prob.b)
        x = torch.zeros_like(b)
        r = s.solve(b, k=30, restart=30, tol=0.0, gs_iters=2, x_out=x)
        out[(diag, walk)] = (np.asarray(r["H"]).tobytes(), np.asarray(r["res_hist"]).tobytes(), x.cpu().numpy().tobytes())
        s.close()
    assert out[("1", None)] == out[("0", None)] == out[("1", "-1")]


# ------------------------------------------------------------- Algorithm 1 (QR)
def _graded_qr(n, m, kappa, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    Wm, _ = np.linalg.qr(rng.standard_normal((m, m)))
    return (U * np.logspace(0, -np.log10(kappa), m)) @ Wm.T


def _gpu_qr(torch, A, sweeps, pad=6):
    import paper_2205_07805_b200 as P
    n, m = A.shape
    ld = n + (n % 2) + pad
    Ah = np.full((m, ld), np.nan)
    Ah[:, :n] = A.T                                # column-major, NaN padding never read
    Ad = _dev(torch, Ah.reshape(-1))
    Qd = torch.full((m * ld,), float("nan"), dtype=torch.float64, device="cuda")
    Rd = torch.full((m * m,), float("nan"), dtype=torch.float64, device="cuda")
    red = P.igs_qr(n, m, Ad, ld, Qd, ld, Rd, sweeps)
    Q = Qd.cpu().numpy().reshape(m, ld)[:, :n].T
    R = Rd.cpu().numpy().reshape(m, m).T
    assert np.array_equal(Ad.cpu().numpy().reshape(m, ld)[:, :n], A.T)   # A untouched
    return Q, R, red


@pytest.mark.parametrize("sweeps", [1, 2])
@pytest.mark.parametrize("shape", [(7, 3), (5000, 40), (70001, 12), (3000, 1)])
def test_igs_qr_vs_oracle(torch_cuda, sweeps, shape):
    n, m = shape
    A = np.random.default_rng(n + m).standard_normal((n, m))
    Q, R, red = _gpu_qr(torch_cuda, A, sweeps)
    Qo, Ro, _, led = oracle.igs_qr(A, sweeps)
    # one (two) reductions per column, + the drain reduction that normalises the last column
    assert red == int(led.sum()) + (m >= 2)
    tol = 1e-12 * np.sqrt(n)
    assert np.abs(R - Ro).max() <= tol * np.abs(Ro).max()
    assert np.abs(Q - Qo).max() <= tol
    assert np.array_equal(np.tril(R, -1), np.zeros((m, m)))
    assert np.linalg.norm(A - Q @ R) <= 1e-14 * np.sqrt(n) * np.linalg.norm(A)
    assert np.linalg.norm(np.eye(m) - Q.T @ Q) <= 1e-13


def test_igs_qr_graded_kappa(torch_cuda):
    # P:792-797 (two sweeps: O(eps)) and P:697-704 (one sweep: O(eps) kappa), on the device
    A = _graded_qr(20000, 30, 1e10, 11)
    kappa = np.linalg.cond(A)
    Q2, R2, _ = _gpu_qr(torch_cuda, A, 2)
    Q1, R1, _ = _gpu_qr(torch_cuda, A, 1)
    loo2 = np.linalg.norm(np.eye(30) - Q2.T @ Q2)
    loo1 = np.linalg.norm(np.eye(30) - Q1.T @ Q1)
    assert loo2 <= 1e-13
    assert loo1 <= 10 * EPS * kappa and loo1 >= 1e3 * loo2
    Qo, Ro, _, _ = oracle.igs_qr(A, 2)
    assert np.abs(R2 - Ro).max() <= 1e-11 * np.abs(Ro).max()
    for Q, R in ((Q1, R1), (Q2, R2)):
        assert np.linalg.norm(A - Q @ R) <= 1e-13 * np.linalg.norm(A)


def test_igs_qr_dependent_column_fails_loudly(torch_cuda):
    import paper_2205_07805_b200 as P
    A = np.random.default_rng(3).standard_normal((1000, 4))
    A[:, 2] = 0.0
    with pytest.raises(P.IgsError):
        _gpu_qr(torch_cuda, A, 2)


# ------------------------------------------------------------- basis diagnostics (NEXT-4)
def _normalized_graded(n, c, kappa, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, c)))
    Wm, _ = np.linalg.qr(rng.standard_normal((c, c)))
    V = (U * np.logspace(0, -np.log10(kappa), c)) @ Wm.T
    return V / np.linalg.norm(V, axis=0)


@pytest.mark.parametrize("case", ["orth", "graded", "graded_odd", "repeated", "one", "wide"])
def test_basis_diag_vs_oracle(torch_cuda, case):
    """igs_op_basis_diag: [||I - V^T V||_F, ||S||_2, sigma_min(V)] on the same V as the
    oracle's definitions."""
    import paper_2205_07805_b200 as P
    rng = np.random.default_rng(len(case))
    n = 5003
    if case == "orth":
        V, _ = np.linalg.qr(rng.standard_normal((n, 40)))
    elif case == "graded":
        V = _normalized_graded(n, 30, 1e3, 1)
    elif case == "graded_odd":
        V = _normalized_graded(n, 31, 1e5, 2)
    elif case == "repeated":
        Q, _ = np.linalg.qr(rng.standard_normal((n, 12)))
        V = np.column_stack([Q, Q[:, 3]])
    elif case == "one":
        V = rng.standard_normal((n, 1)); V /= np.linalg.norm(V)
    else:
        V, _ = np.linalg.qr(rng.standard_normal((n, 257)))
        V[:, 200] = (V[:, 200] + 1e-3 * V[:, 10]) / np.linalg.norm(V[:, 200] + 1e-3 * V[:, 10])
    c = V.shape[1]
    ld = n + 5
    Vh = np.zeros((c, ld)); Vh[:, :n] = V.T
    Vd = _dev(torch_cuda, Vh.reshape(-1))
    loo, s2, smin = P.igs_op_basis_diag(n, c, Vd, ld)
    lo = oracle.loss_of_orthogonality(V)
    so = oracle.S_norm(V, c)
    mo = oracle.sigma_min(V, c)
    # G = V^T V entries carry ~sqrt(n) eps of reduction-order noise: eps-level values agree
    # to an absolute 1e-12, larger ones to 1e-10 relative
    assert abs(loo - lo) <= 1e-10 * lo + 1e-12, (loo, lo)
    assert abs(s2 - so) <= 1e-10 * so + 1e-12, (s2, so)
    # sigma_min through the Gram matrix: absolute accuracy ~ c eps / sigma_min (reading R23)
    assert abs(smin - mo) <= 1e-10 * mo + 64 * c * EPS / max(mo, 1e-8), (smin, mo)
    if case == "repeated":
        assert abs(s2 - 1.0) <= 1e-10 and smin <= 1e-7

