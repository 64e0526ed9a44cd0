"""The G > 1 code paths on ONE B200 (the pool gives one GPU; NCCL cannot put two ranks on one
device, and ranks whose kernels wait on each other must not share one).

* Halo: `igs_create_virtual` builds the G per-rank contexts of a
  row-block partition on one device with the same halo plan igs_create computes at G > 1;
  `igs_virtual_spmv` runs every rank's pack kernel, then each rank's SpMV exactly as the solve
  does at G > 1 (interior rows with the ghost-aware SELL kernel while the ghosts arrive, the
  boundary rows by the row-list kernel after them) with device copies in place of
  ncclSend/ncclRecv.  Row sums are left to right with separate multiply and add on both sides,
  so the result must equal oracle.spmv (P:1055-1059 Step 4, A u) bit for bit.
* Failure handling: the fused exchange's device barrier timeout and the host
  deadline, on 1-rank communicators, turn a hang into IGS_ERR_NCCL.
* CUDA-graph capture with collectives inside (the G > 1 launch path of small slabs), on 1-rank
  communicators: the same bits as the plain path.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2205_07805_b200 as P
    P.lib()
    return P


def _plane_bounds(N, G):
    planes = [N * q // G for q in range(G + 1)]
    return np.array([p * N * N for p in planes], dtype=np.int64)


def _virtual_spmv(P, A, bounds, x, b=None):
    import torch
    g = P.igs.VirtualGroup(A, bounds)
    try:
        xs = [torch.from_numpy(np.ascontiguousarray(x[bounds[r]:bounds[r + 1]])).cuda() for r in range(g.G)]
        ys = [torch.full((int(bounds[r + 1] - bounds[r]),), np.nan, dtype=torch.float64, device="cuda")
              for r in range(g.G)]
        bs = None
        if b is not None:
            bs = [torch.from_numpy(np.ascontiguousarray(b[bounds[r]:bounds[r + 1]])).cuda() for r in range(g.G)]
        g.spmv(xs, ys, bs)
        y = np.concatenate([t.cpu().numpy() for t in ys])
        return y, g.stats()
    finally:
        g.close()


@pytest.mark.parametrize("sell", ["1", "0"])
@pytest.mark.parametrize("split", ["planes2", "planes3", "planes8", "ragged3", "ragged5"])
def test_virtual_halo_spmv_c4_24(P, split, sell, monkeypatch):
    """c4's operator at 24^3 (n = 13824) cut into G row blocks: z-slabs (G = 2, 3, 8 -- the
    bench's partition) and ragged blocks that cut planes (every rank needs ghosts from up to
    two owners per side).  IGS_SELL=0: the CSR kernels with ghost columns and no split."""
    monkeypatch.setenv("IGS_SELL", sell)
    N = 24
    prob = W.config("c4", N=N)
    n = N ** 3
    if split.startswith("planes"):
        bounds = _plane_bounds(N, int(split[6:]))
    else:
        G = int(split[6:])
        rng = np.random.default_rng(G)
        cuts = np.sort(rng.choice(np.arange(1, n), G - 1, replace=False))
        bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    x = np.random.default_rng(5).standard_normal(n)
    y, st = _virtual_spmv(P, prob.A, bounds, x)
    ref = oracle.spmv(prob.A, x)
    assert y.tobytes() == ref.tobytes(), np.max(np.abs(y - ref))
    # residual mode (r = b - A x at cycle start): one subtraction after the row sum
    yr, _ = _virtual_spmv(P, prob.A, bounds, x, prob.b)
    assert yr.tobytes() == (prob.b - ref).tobytes()
    G = len(bounds) - 1
    if split.startswith("planes"):  # one halo message per neighbour slab
        assert [s["halo_msgs"] for s in st] == [1] + [2] * (G - 2) + [1]


def test_virtual_halo_spmv_random_sparse(P):
    """A random non-symmetric sparse matrix (3-12 entries per row, columns anywhere): ghosts
    from every rank, uneven blocks, one empty block."""
    rng = np.random.default_rng(11)
    n = 5000
    rows, cols = [], []
    for i in range(n):
        c = np.unique(np.concatenate([[i], rng.choice(n, rng.integers(2, 12), replace=False)]))
        rows.append(np.full(len(c), i)), cols.append(c)
    cols = np.concatenate(cols).astype(np.int32)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    A = W.Csr(n, n, 0, rowptr, cols, rng.standard_normal(len(cols)))
    bounds = np.array([0, 700, 700, 2500, 2600, 5000], dtype=np.int64)
    x = rng.standard_normal(n)
    y, _ = _virtual_spmv(P, A, bounds, x)
    assert y.tobytes() == oracle.spmv(A, x).tobytes()


@pytest.mark.parametrize("cfg,G", [("c4", 8), ("c4", 2), ("c5", 8)])
def test_virtual_halo_spmv_full_size(P, cfg, G):
    """BASELINE configs at full size, partitioned as bench.py / SURVEY §8(e) shard them:
    c4 (256^3) into 8 z-slabs of 32 planes (2.1M rows each) and into 2 slabs; c5 (512^3,
    int64 columns) into 8 slabs of 64 planes (16.8M rows each).  Every row bitwise against the
    oracle's SpMV."""
    prob = W.config(cfg)
    N = 256 if cfg == "c4" else 512
    bounds = _plane_bounds(N, G)
    x = np.random.default_rng(7).standard_normal(N ** 3)
    y, st = _virtual_spmv(P, prob.A, bounds, x)
    ref = oracle.spmv(prob.A, x)
    assert y.tobytes() == ref.tobytes(), np.max(np.abs(y - ref))
    assert [s["halo_msgs"] for s in st] == [1] + [2] * (G - 2) + [1]


def test_virtual_contexts_reject_solve(P):
    import torch
    prob = W.config("c4", N=12)
    g = P.igs.VirtualGroup(prob.A, _plane_bounds(12, 2))
    try:
        res = P.igs.igs_result()
        x = torch.empty(g.bounds[1], dtype=torch.float64, device="cuda")
        res.x = x.data_ptr()
        b = torch.ones(g.bounds[1], dtype=torch.float64, device="cuda")
        with pytest.raises(P.IgsError) as e:
            P.igs.igs_solve(g.ctxs[0], P.igs.IGS_MEM_DEVICE, b, None, 10, 0, 0.0, 2, res)
        assert e.value.status == P.igs.IGS_ERR_ARG
    finally:
        g.close()


# ------------------------------------------------------------------ failure handling
def test_exchange_barrier_timeout_fails_instead_of_hanging(P, monkeypatch):
    """IGS_TEST_XCHG_STALL=c: exchange number c waits for a peer epoch that never arrives --
    what a rank sees when a peer died.  With a 1 s bound the solve must return IGS_ERR_NCCL
    (communicator aborted) within seconds, later solves IGS_ERR_STATE, and destroy works."""
    import time
    import torch
    monkeypatch.setenv("IGS_XCHG", "1")
    monkeypatch.setenv("IGS_PERSIST", "0")
    monkeypatch.setenv("IGS_TEST_XCHG_STALL", "7")
    prob = W.config("c3", N=64)
    b = torch.from_numpy(prob.b).cuda()
    s = P.Solver(prob.A)
    s.set_timeout(1.0)
    t0 = time.time()
    with pytest.raises(P.IgsError) as e:
        s.solve(b, k=40, gs_iters=2)
    assert e.value.status == P.igs.IGS_ERR_NCCL and "barrier timeout" in str(e.value), str(e.value)
    assert time.time() - t0 < 60
    with pytest.raises(P.IgsError) as e2:
        s.solve(b, k=40, gs_iters=2)
    assert e2.value.status == P.igs.IGS_ERR_STATE
    s.close()


def test_host_deadline_aborts_communicator(P, monkeypatch):
    """A host wait that outlasts the deadline (a collective that never completes looks like
    this) aborts the communicator: IGS_ERR_NCCL with 'timeout', then IGS_ERR_STATE."""
    import torch
    monkeypatch.setenv("IGS_FORCE_NCCL", "1")
    monkeypatch.setenv("IGS_PERSIST", "0")
    prob = W.config("c3", N=512)
    b = torch.from_numpy(prob.b).cuda()
    s = P.Solver(prob.A)
    s.solve(b, k=20, gs_iters=2)          # warm-up with the default deadline
    s.set_timeout(1e-4)                    # far below one cycle (~ms)
    with pytest.raises(P.IgsError) as e:
        s.solve(b, k=100, gs_iters=2)
    assert e.value.status == P.igs.IGS_ERR_NCCL and "timeout" in str(e.value), str(e.value)
    with pytest.raises(P.IgsError) as e2:
        s.solve(b, k=10, gs_iters=2)
    assert e2.value.status == P.igs.IGS_ERR_STATE
    s.close()


# ------------------------------------------------ graphs with collectives inside (G > 1 path)
@pytest.mark.parametrize("mode", ["xchg", "nccl"])
@pytest.mark.parametrize("alg", ["igs2", "igs1", "igs2_two", "mgs"])
def test_graph_capture_with_collectives_one_rank(P, mode, alg, monkeypatch):
    """Small slabs at G > 1 replay whole cycles from CUDA graphs with the exchange kernels /
    ncclAllReduce captured inside.  On a 1-rank communicator: bitwise the graph-less plain
    path, with a convergence stop inside a cycle (the nodes after it run as no-ops while the
    collectives still run)."""
    import torch
    prob = W.config("c3", N=96)
    b = torch.from_numpy(prob.b).cuda()
    k, restart = (90, 40) if alg != "mgs" else (40, 20)
    outs = {}
    for variant in ("comm", "plain"):
        monkeypatch.setenv("IGS_PERSIST", "0")
        monkeypatch.setenv("IGS_XCHG", "1" if variant == "comm" and mode == "xchg" else "0")
        monkeypatch.setenv("IGS_FORCE_NCCL", "1" if variant == "comm" and mode == "nccl" else "0")
        monkeypatch.setenv("IGS_GRAPHS", "1" if variant == "comm" else "0")
        s = P.Solver(prob.A)
        outs[variant] = [s.solve(b, k=k, restart=restart, tol=1e-9, algorithm=alg) for _ in range(2)]
        s.close()
    for g, u in zip(outs["comm"], outs["plain"]):
        assert g["iters"] == u["iters"] and g["term"] == u["term"] and g["cycles"] == u["cycles"]
        assert g["H"].tobytes() == u["H"].tobytes()
        assert g["x"].cpu().numpy().tobytes() == u["x"].cpu().numpy().tobytes()
        assert g["allreduces"] >= g["reductions"] > 0


@pytest.mark.parametrize("mode", ["xchg", "nccl"])
def test_graph_capture_split_spmv_one_rank(P, mode, monkeypatch):
    """The G > 1 SpMV split inside a captured cycle: IGS_TEST_BND_EVERY routes every 7th row
    through the boundary pass, so each SpMV forks to the halo stream and joins back (event
    record / wait inside the capture) around the interior rows, with the exchange kernels or
    ncclAllReduce captured too (1-rank communicator).  Bitwise the plain graph-less path."""
    import torch
    prob = W.config("c4", N=40)
    b = torch.from_numpy(prob.b).cuda()
    outs = {}
    for variant in ("comm", "plain"):
        monkeypatch.setenv("IGS_PERSIST", "0")
        monkeypatch.setenv("IGS_XCHG", "1" if variant == "comm" and mode == "xchg" else "0")
        monkeypatch.setenv("IGS_FORCE_NCCL", "1" if variant == "comm" and mode == "nccl" else "0")
        monkeypatch.setenv("IGS_GRAPHS", "1" if variant == "comm" else "0")
        monkeypatch.setenv("IGS_TEST_BND_EVERY", "7" if variant == "comm" else "0")
        s = P.Solver(prob.A)
        outs[variant] = s.solve(b, k=120, restart=50, tol=1e-11, algorithm="igs2")
        info = s.info()
        s.close()
        if variant == "comm":
            assert info["graph_launches"] > 0 and info["n_bnd"] > 0, info
    g, u = outs["comm"], outs["plain"]
    assert g["iters"] == u["iters"] and g["cycles"] == u["cycles"] and g["H"].tobytes() == u["H"].tobytes()
    assert g["x"].cpu().numpy().tobytes() == u["x"].cpu().numpy().tobytes()


# ------------------------------------------------------------------ G > 1 solve, one device
def _virtual_solve(P, prob, bounds, **kw):
    import torch
    g = P.igs.VirtualGroup(prob.A, bounds)
    try:
        bs = [torch.from_numpy(np.ascontiguousarray(prob.b[bounds[r]:bounds[r + 1]])).cuda() for r in range(g.G)]
        xs = [torch.full((int(bounds[r + 1] - bounds[r]),), np.nan, dtype=torch.float64, device="cuda")
              for r in range(g.G)]
        res = g.solve(bs, xs, **kw)
        x = np.concatenate([t.cpu().numpy() for t in xs])
        return res, x, g.stats()
    finally:
        g.close()


def _cols_diff(Hg, Ho, rh, ncols=30):
    c = 0
    while c < min(ncols, Ho.shape[1]) and (c + 1 >= len(rh) or rh[c + 1] > 1e-8):
        c += 1
    return oracle.column_normwise_diff(Hg, Ho, max(c, 1))


@pytest.mark.parametrize("alg", ["igs2", "igs1", "igs2_two", "mgs"])
@pytest.mark.parametrize("split", ["planes2", "planes3", "ragged4"])
def test_virtual_solve_vs_oracle(P, split, alg):
    """The G > 1 solve with the product's own per-rank control flow on one
    device (igs_virtual_solve: row-block slabs, the halo overlapped with the interior rows,
    one cross-rank sum per reduction with the transports emulated): c4's operator at 16^3,
    GMRES(30) to 1e-10 over several cycles.  Against the oracle on the whole matrix: the
    Hessenberg matrix of the first cycle column-normwise (R9), the residual history, the
    iteration / cycle counts and x; across ranks: the replicated state (H, residual history)
    bit for bit, and exactly one cross-rank sum per reduction."""
    N = 16
    prob = W.config("c4", N=N)
    n = N ** 3
    if split.startswith("planes"):
        bounds = _plane_bounds(N, int(split[6:]))
    else:
        rng = np.random.default_rng(9)
        cuts = np.sort(rng.choice(np.arange(1, n), 3, replace=False))
        bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    k, restart, tol = 400, 30, 1e-10
    res, x, st = _virtual_solve(P, prob, bounds, k=k, restart=restart, tol=tol, algorithm=alg)
    o = oracle.gmres(prob.A, prob.b, k, restart=restart, tol=tol, variant=alg, dot_block=4096)
    r0 = res[0]
    for r in res[1:]:   # replicated small state: identical bits on every rank
        assert r["H"].tobytes() == r0["H"].tobytes() and r["res_hist"].tobytes() == r0["res_hist"].tobytes()
        assert (r["iters"], r["cycles"], r["term"]) == (r0["iters"], r0["cycles"], r0["term"])
    assert r0["term"] == o["term"] == "converged"
    assert abs(r0["iters"] - o["iters"]) <= 1 and r0["cycles"] == o["cycles"], (r0["iters"], o["iters"])
    d = _cols_diff(r0["H"], o["H"], o["res_hist"])
    assert d <= 1e-10 or (alg in ("igs1", "mgs") and d <= 1e-8), d
    m = min(len(r0["res_hist"]), len(o["res_hist"]))
    np.testing.assert_allclose(r0["res_hist"][:m], o["res_hist"][:m], rtol=1e-6)
    assert r0["true_relres"] <= 1e-10
    np.testing.assert_allclose(x, o["x"], rtol=0, atol=1e-8 * np.max(np.abs(o["x"])))
    # ledger: IGS(1) / Alg. 3 one cross-rank sum per iteration, Alg. 2 two, MGS j+2 per column
    # (+ ||b||, the residual at each cycle start and the final one, the priming h per cycle)
    if alg in ("igs1", "igs2"):
        assert r0["reductions"] <= r0["iters"] + 4 * r0["cycles"] + 4, (r0["reductions"], r0["iters"])
    for s in st:
        assert s["allreduces"] >= r0["reductions"]


def test_virtual_solve_c4_slabs_loo(P):
    """c4 at 32^3 in 8 z-slabs of 4 planes (every interior rank has two neighbours),
    Alg. 3, one unrestarted cycle of 60 iterations with the LOO diagnostic (its Gram summed
    across ranks like the dots): H over 30 columns (R9) and ||I - V^T V||_F within 10x
     of the oracle's."""
    N = 32
    prob = W.config("c4", N=N)
    bounds = _plane_bounds(N, 8)
    res, x, st = _virtual_solve(P, prob, bounds, k=60, restart=0, tol=0.0, algorithm="igs2", want_loo=True)
    o = oracle.gmres(prob.A, prob.b, 60, variant="igs2", dot_block=4096, want_V=True)
    r0 = res[0]
    assert all(r["H"].tobytes() == r0["H"].tobytes() and r["loo"] == r0["loo"] for r in res)
    assert r0["iters"] == o["iters"] == 60
    assert _cols_diff(r0["H"], o["H"], o["res_hist"]) <= 1e-10
    lo = oracle.loss_of_orthogonality(o["V"][:, :o["basis_cols"]])
    assert (r0["loo"] < 1e-12 and lo < 1e-12) or lo / 10 <= r0["loo"] <= 10 * lo, (r0["loo"], lo)
    assert all(s["halo_msgs"] > 0 for s in st)
