"""Pins for the oracle's GMRES variants (CPU only).

Each test ties the oracle to something other than itself: dense LU, scipy's GMRES,
the Arnoldi relation, orthogonality bounds of the paper (P:697-704, P:792-797,
P:1158-1164), beta*kappa(B_k)=O(1), the paper's printed Section-5 behaviour
(tests/golden/paper_values.json), and exact-arithmetic termination facts.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
EPS = np.finfo(float).eps
ALL = ["mgs", "igs1", "igs2_two", "igs2"]
TWO_SWEEP = ["igs2_two", "igs2"]


@pytest.fixture(scope="module")
def c1_runs():
    P = W.config("c1")
    return P, {v: oracle.gmres(P.A, P.b, 60, variant=v, want_V=True, want_L=True) for v in ALL}


@pytest.mark.parametrize("v", ALL)
def test_identity_converges_in_one_iteration(v):
    # A = I -> one iteration, x = b (happy breakdown after column 0)
    A = W.diag_csr(np.ones(12)); b = np.arange(1.0, 13.0)
    o = oracle.gmres(A, b, 5, variant=v)
    assert o["iters"] == 1 and o["term"] == "breakdown"
    np.testing.assert_allclose(o["x"], b, rtol=1e-15)


@pytest.mark.parametrize("v", ALL)
def test_diagonal_terminates_at_number_of_distinct_eigenvalues(v):
    # exact arithmetic: K_j(A, b) has dimension = number of distinct eigenvalues (5)
    d = np.tile(np.arange(1.0, 6.0), 10)
    A = W.diag_csr(d); b = np.ones(50)
    o = oracle.gmres(A, b, 40, variant=v)
    assert o["term"] == "breakdown"
    # two sweeps detect the invariant subspace at column 4 (5 iterations); one sweep and
    # MGS see a subdiagonal ~3e-14 relative (above reading R12's 64 eps) and stop one later
    assert o["iters"] == 5 if v in TWO_SWEEP else o["iters"] in (5, 6)
    np.testing.assert_allclose(o["x"], b / d, rtol=1e-14)


@pytest.mark.parametrize("v", ALL)
@pytest.mark.parametrize("n", [20, 45])
def test_dense_lu_small_systems(v, n):
    rng = np.random.default_rng(n)
    D = np.eye(n) * 4 + rng.uniform(-1, 1, (n, n))
    A = W.dense_to_csr(D)
    b = rng.standard_normal(n)
    o = oracle.gmres(A, b, n, tol=1e-14, variant=v)
    xs = np.linalg.solve(D, b)
    kappa = np.linalg.cond(D)
    assert np.linalg.norm(o["x"] - xs) <= 1e3 * EPS * kappa * np.linalg.norm(xs)


@pytest.mark.parametrize("v", ALL)
def test_arnoldi_relation_c1(c1_runs, v):
    P, runs = c1_runs
    o = runs[v]
    rel = oracle.arnoldi_relation(P.A, o["V"], o["H"], o["h_cols"])
    assert rel <= 1000 * P.A.n_rows * EPS
    assert rel <= 1e-15                             # observed 4e-17..7e-17


@pytest.mark.parametrize("v", ALL)
def test_arnoldi_relation_simoncini(v):
    A, b = W.simoncini(100, 0)
    o = oracle.gmres(A, b, 60, variant=v, want_V=True)
    assert oracle.arnoldi_relation(A, o["V"], o["H"], 60) <= 1e-15


def test_orthogonality_two_sweeps_c1(c1_runs):
    _, runs = c1_runs
    for v in TWO_SWEEP:
        o = runs[v]
        assert oracle.loss_of_orthogonality(o["V"][:, :o["basis_cols"]]) <= 1e-13   # O(eps)


def test_orthogonality_one_sweep_and_mgs_follow_eps_kappa(c1_runs):
    # one sweep / MGS: ||I - V^T V|| <~ c eps kappa(B_k)
    P, runs = c1_runs
    for v in ("mgs", "igs1"):
        o = runs[v]
        p = o["h_cols"]
        loo = oracle.loss_of_orthogonality(o["V"][:, :p])
        kap = oracle.kappa_Bk(P.A, P.b, o["V"], p)
        assert loo <= 10 * EPS * kap
        assert loo >= 1e3 * oracle.loss_of_orthogonality(runs["igs2"]["V"][:, :p])


def test_beta_kappa_is_order_one(c1_runs):
    # beta(x_k) kappa(B_k) = O(1); band of reading R13
    P, _ = c1_runs
    normA = oracle.norm2_estimate(P.A)
    for v in ALL:
        for k in (10, 20, 30, 45):
            o = oracle.gmres(P.A, P.b, k, variant=v, want_V=True)
            beta = oracle.backward_error(P.A, P.b, o["x"], normA)
            if beta > 1e3 * EPS:
                kap = oracle.kappa_Bk(P.A, P.b, o["V"], k)
                assert 0.1 <= beta * kap <= 10, (v, k, beta, kap)


def test_cross_variant_hessenberg_agreement(c1_runs):
    _, runs = c1_runs
    ref = runs["igs2_two"]["H"]
    for v in ALL:
        assert oracle.column_normwise_diff(runs[v]["H"], ref, 30) <= 1e-10


@pytest.mark.parametrize("mk", ["c1", "simoncini"])
def test_lagged_norm_agrees_with_explicit_norm(mk):
    # "diagonal elements R_kk computed with the lagged norm agree closely"
    if mk == "c1":
        P = W.config("c1"); A, b, k = P.A, P.b, 60
    else:
        (A, b), k = W.simoncini(100, 1), 98
    H2 = oracle.gmres(A, b, k, variant="igs2_two")["H"]
    H3 = oracle.gmres(A, b, k, variant="igs2")["H"]
    s2 = np.array([H2[j + 1, j] for j in range(k)])
    s3 = np.array([H3[j + 1, j] for j in range(k)])
    assert np.max(np.abs(s2 - s3) / s2) <= 1e-12


@pytest.mark.parametrize("v", ["igs1", "igs2", "igs2_two"])
@pytest.mark.parametrize("N", [16, 32])
def test_restart_counts_match_scipy(v, N):
    # library routine: scipy GMRES(100) on the c4 operator; inner iteration counts and the
    # final true residual must agree (restart semantics of SURVEY §8(c) "Driver")
    import scipy.sparse.linalg as sla
    P = W.config("c4", N=N)
    cnt = [0]
    x, info = sla.gmres(P.A.to_scipy(), P.b, rtol=1e-12, restart=100, maxiter=100,
                        callback=lambda _: cnt.__setitem__(0, cnt[0] + 1), callback_type="pr_norm")
    o = oracle.gmres(P.A, P.b, 3000, restart=100, tol=1e-12, variant=v)
    assert info == 0 and o["term"] == "converged"
    assert o["iters"] == cnt[0]
    ref = np.linalg.norm(P.b - P.A.to_scipy() @ x) / np.linalg.norm(P.b)
    assert o["true_relres"] <= 1e-12 and abs(o["true_relres"] - ref) <= 0.05 * ref


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_simoncini_mgs_stagnates_igs2_does_not(seed):
    g = GOLD["simoncini"]
    A, b = W.simoncini(100, seed)
    # power iteration with S:79's stopping rule (rel. change 1e-4) is within 1% here
    assert oracle.norm2_estimate(A) == pytest.approx(g["norm2_A"], rel=1e-2)
    assert np.linalg.cond(A.to_dense()) == pytest.approx(g["kappa_A"], rel=1e-12)
    mgs = oracle.gmres(A, b, 98, variant="mgs", want_V=True)
    it = g["mgs_stagnation_after_iteration"]
    r = mgs["res_hist"]
    # MGS: stagnates around 1e-12 after iteration 75, ||S_k|| -> 1
    assert r[it:].min() >= 0.1 * g["mgs_stagnation_level"]
    assert r[it:].max() <= 100 * g["mgs_stagnation_level"]
    assert oracle.S_norm(mgs["V"], 98) >= 0.99
    for v in TWO_SWEEP:
        o = oracle.gmres(A, b, 98, variant=v, want_V=True)
        rr = o["res_hist"]
        assert rr[90] <= 1e-18 and rr[98] <= 1e-24          # continues to decrease
        assert np.all(np.diff(rr) <= 1e-30)                 # monotone
        assert oracle.S_norm(o["V"], 98) <= 1e-12
        assert oracle.loss_of_orthogonality(o["V"][:, :o["basis_cols"]]) <= 1e-13


def test_walker_printed_values():
    g = GOLD["walker"]
    A, b = W.walker(10, g["alpha"])
    D = A.to_dense()
    assert np.linalg.cond(D) == pytest.approx(g["kappa_A"], rel=0.05)
    assert oracle.norm2_estimate(A) == pytest.approx(g["norm2_A"], rel=0.05)
    ev = np.linalg.eigvals(D)
    dep = np.sqrt(np.linalg.norm(D, "fro") ** 2 - np.sum(np.abs(ev) ** 2))   # Henrici
    assert dep == pytest.approx(g["dep_A"], rel=1e-9)
    o = oracle.gmres(A, b, 8, variant="igs2", want_V=True)
    assert oracle.loss_of_orthogonality(o["V"][:, :o["basis_cols"]]) <= 1e-14


def test_embree_printed_values():
    g = GOLD["embree"]
    A, b = W.embree(100, 0.1)
    D = A.to_dense()
    assert np.linalg.norm(D, 2) == pytest.approx(g["norm2_A"], abs=0.05)
    assert np.linalg.cond(D) == pytest.approx(g["kappa_A"], abs=0.05)
    for v in TWO_SWEEP:
        o = oracle.gmres(A, b, 30, tol=1e-12, variant=v)
        assert o["term"] == "converged" and o["iters"] <= g["igs_iterations_to_converge"]


def test_helmert_orthogonality():
    A, b = W.helmert(18)
    D = A.to_dense()
    assert np.linalg.norm(D.T @ D - np.eye(18)) <= 1e-14
    for v in TWO_SWEEP:
        o = oracle.gmres(A, b, 16, variant=v, want_V=True)
        assert oracle.loss_of_orthogonality(o["V"][:, :o["basis_cols"]]) <= 1e-14


def test_ledger_counts(c1_runs):
    g = GOLD["ledger"]
    _, runs = c1_runs
    assert np.all(runs["igs1"]["ledger"] == g["igs1_per_iteration"])
    assert np.all(runs["igs2"]["ledger"] == g["alg3_per_iteration"])
    led2 = runs["igs2_two"]["ledger"]
    assert np.all(led2[:-1] == g["alg2_two_reduce_per_iteration"]) and led2[-1] == 1   # drain
    # MGS: iteration t computes t inner products + 1 norm (k-1 projections + norm)
    np.testing.assert_array_equal(runs["mgs"]["ledger"], np.arange(2, 62))
    for v in ("igs1", "igs2", "igs2_two"):
        assert runs[v]["priming_reductions"] == 2


def test_reduction_order_noise_floor_two_sweeps():
    # reordering only the reductions moves two-sweep H by ~1e-15 normwise
    P = W.config("c1")
    a = oracle.gmres(P.A, P.b, 40, variant="igs2")
    b = oracle.gmres(P.A, P.b, 40, variant="igs2", dot_block=64)
    assert oracle.column_normwise_diff(b["H"], a["H"], 30) <= 1e-13


def test_x0_and_zero_rhs():
    P = W.config("c1")
    o = oracle.gmres(P.A, np.zeros(1000), 10, variant="igs2")
    assert o["term"] == "converged" and o["iters"] == 0 and np.all(o["x"] == 0)
    xs = np.linalg.solve(P.A.to_dense(), P.b)
    o = oracle.gmres(P.A, P.b, 10, tol=1e-10, variant="igs2", x0=xs)
    assert o["iters"] == 0 and o["term"] == "converged"


def test_nonfinite_rejected():
    P = W.config("c1")
    b = P.b.copy(); b[3] = np.nan
    with pytest.raises(ValueError):
        oracle.gmres(P.A, b, 5)
