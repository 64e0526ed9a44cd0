"""The seeded input generators: shapes/nnz of BASELINE.json configs, CSR validity and
bitwise shard consistency (CPU only)."""
import numpy as np
import pytest

import workloads as W


def _valid(A):
    assert A.rowptr[0] == 0 and np.all(np.diff(A.rowptr) >= 0) and A.rowptr[-1] == A.colind.size
    for i in range(0, A.n_rows, max(1, A.n_rows // 50)):
        c = A.colind[A.rowptr[i]:A.rowptr[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < A.n_cols


@pytest.mark.parametrize("name,nnz", [("c1", 2998), ("c2", 2001000)])
def test_small_configs(name, nnz):
    P = W.config(name)
    assert P.A.nnz == nnz
    _valid(P.A)


def test_stencil_nnz_formula():
    # 2D: 5N^2 - 4N (c3: N=1024 -> 5,238,784); 3D: 7N^3 - 6N^2 (c4: 117,047,296; c5: 937,951,232)
    for N in (5, 17, 64):
        assert W.stencil_csr(N, 2, W.C3_BETA).nnz == 5 * N * N - 4 * N
        assert W.stencil_csr(N, 3, W.C4_BETA).nnz == 7 * N ** 3 - 6 * N ** 2
    assert 5 * 1024 ** 2 - 4 * 1024 == 5238784
    assert 7 * 256 ** 3 - 6 * 256 ** 2 == 117047296
    assert 7 * 512 ** 3 - 6 * 512 ** 2 == 937951232


def test_stencil_entries_against_pde_coefficients():
    N = 9
    A = W.stencil_csr(N, 3, W.C4_BETA).to_dense()
    h = 1.0 / (N + 1)
    i, j, l = 4, 3, 5
    r = i + N * j + N * N * l
    assert A[r, r] == 6.0
    for d, (off, bt) in enumerate(zip((1, N, N * N), W.C4_BETA)):
        assert A[r, r - off] == -1.0 - (bt * h) / 2.0      # upwind side
        assert A[r, r + off] == -1.0 + (bt * h) / 2.0
    assert np.count_nonzero(A[r]) == 7


@pytest.mark.parametrize("G", [2, 3, 4])
def test_shards_are_bitwise_rows_of_the_whole(G):
    N = 12
    full = W.stencil_csr(N, 3, W.C4_BETA)
    n = N ** 3
    bounds = [n * g // G for g in range(G + 1)]
    for g in range(G):
        s = W.stencil_csr(N, 3, W.C4_BETA, bounds[g], bounds[g + 1])
        a, b = full.rowptr[bounds[g]], full.rowptr[bounds[g + 1]]
        assert np.array_equal(s.colind, full.colind[a:b])
        assert s.values.tobytes() == full.values[a:b].tobytes()
        assert np.array_equal(s.rowptr, full.rowptr[bounds[g]:bounds[g + 1] + 1] - a)


def test_c4_rhs_seed_and_int64_variant():
    P = W.config("c4", N=8)
    assert np.array_equal(P.b, np.random.default_rng(3).uniform(0.0, 1.0, 512))
    A64 = W.stencil_csr(8, 3, W.C5_BETA, index_bits=64)
    assert A64.colind.dtype == np.int64 and A64.index_bits == 64
