"""Randomized GPU-vs-oracle sweep: random sparse non-symmetric matrices (row lengths 1..40,
a random band plus scattered entries, diagonally dominant), random sizes across the
persistent-kernel, graph and per-kernel paths, random k / restart / tolerance, all four
algorithms.  Seeded: every case is reproducible from its id."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
ALGS = ["igs2", "igs1", "igs2_two", "mgs"]


def random_csr(n, rng, wide=False):
    rows, cols, vals = [], [], []
    band = int(rng.integers(1, 6))
    extra = 60 if wide else 8   # wide: ~30 nnz/row on average -> the vector-CSR SpMV
    for i in range(n):
        js = set(range(max(0, i - band), min(n, i + band + 1)))
        js.update(int(j) for j in rng.integers(0, n, int(rng.integers(0, extra))))
        js = sorted(js)
        v = rng.standard_normal(len(js)) * 0.3
        v[js.index(i)] = 2.0 + len(js) * 0.3 + rng.uniform(0, 1)
        rows.append(len(js)); cols.extend(js); vals.extend(v)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(rows, out=rowptr[1:])
    return W.Csr(n, n, 0, rowptr, np.asarray(cols, dtype=np.int32), np.asarray(vals))


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2205_07805_b200 as P
    P.lib()
    return P


@pytest.mark.parametrize("case", range(64))
def test_random_systems_vs_oracle(P, case):
    import torch
    rng = np.random.default_rng(1000 + case)
    n = int(rng.choice([60, 300, 1500, 5000, 20000, 70000, 150000]))
    A = random_csr(min(n, 20000) if case % 5 == 4 else n, rng, wide=case % 5 == 4)
    n = A.n_rows
    b = rng.standard_normal(n)
    alg = ALGS[case % 4]
    k = int(rng.integers(5, 90 if alg != "mgs" else 40))
    restart = int(rng.choice([0, max(2, k // 3), k // 2 + 1]))
    tol = float(rng.choice([0.0, 1e-8, 1e-11]))
    s = P.Solver(A)
    g = s.solve(torch.from_numpy(b).cuda(), k=k, restart=restart, tol=tol, algorithm=alg)
    s.close()
    o = oracle.gmres(A, b, k, restart=restart, tol=tol, variant=alg, dot_block=4096)
    assert g["term"] == o["term"], (g["term"], o["term"])
    assert abs(g["iters"] - o["iters"]) <= 1 and g["cycles"] in (o["cycles"], o["cycles"] + 1, o["cycles"] - 1)
    if g["iters"] == o["iters"]:
        scale = np.abs(o["x"]).max()
        assert np.abs(g["x"].cpu().numpy() - o["x"]).max() <= 1e-8 * scale, alg
        m = min(len(g["res_hist"]), len(o["res_hist"]))
        np.testing.assert_allclose(g["res_hist"][:m], o["res_hist"][:m], rtol=1e-5, atol=1e-13)
    assert g["true_relres"] <= max(10 * o["true_relres"], 1e-13) or g["true_relres"] <= tol
