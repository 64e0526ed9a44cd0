"""Host-only SELL-32 layout (igs_plan_sell, the arrays igs_create uploads for the SpMV of
P:1059 Step 4) on the CPU: the arrays must decode back to the input CSR entry for entry, in
order; the slice classification must be the one the matrix implies; a numpy SpMV that walks
the arrays the way the kernels do (list positions in order, separate multiply and add) must
equal the oracle's row loop bit for bit."""
import numpy as np
import pytest

import oracle
import workloads as W
import paper_2205_07805_b200 as P


def _banded(n, offs, drop, rng, scatter_rows=0):
    cols = []
    for r in range(n):
        c = np.array([r + o for o in offs if 0 <= r + o < n and rng.random() >= drop], dtype=np.int64)
        if r < scatter_rows:
            c = np.union1d(c, rng.integers(0, n, 3))
        cols.append(c)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([c.size for c in cols], out=rowptr[1:])
    colind = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    return W.Csr(n, n, 0, rowptr, colind.astype(np.int64), rng.standard_normal(colind.size))


def _decode(n, S):
    """rows -> (columns, values) from the SELL arrays, the way sell_row reads them."""
    out = []
    for r in range(n):
        s, l = r >> 5, r & 31
        if S["len"][r] == 255:
            out.append(None)
            continue
        if S["cptr"][s + 1] == S["cptr"][s]:          # diagonal slice: list positions in order
            js = [j for j in range(8) if (S["mask"][r] >> j) & 1]
            cols = [r + int(S["diag"][8 * s + j]) for j in js]
            vals = [S["val"][S["ptr"][s] + 32 * j + l] for j in js]
        else:                                          # explicit slice: entry index
            ks = range(int(S["len"][r]))
            cols = [int(S["col"][S["cptr"][s] + 32 * k + l]) for k in ks]
            vals = [S["val"][S["ptr"][s] + 32 * k + l] for k in ks]
        out.append((cols, vals))
    return out


CASES = {
    "band7_masked": lambda rng: (_banded(1013, [-70, -7, -1, 0, 1, 7, 70], 0.2, rng), "all"),
    "band9": lambda rng: (_banded(700, [-90, -40, -9, -1, 0, 1, 9, 40, 90], 0.2, rng), "ends"),
    "band8_mixed": lambda rng: (_banded(901, [-300, -17, -1, 0, 1, 17, 300, 301], 0.1, rng, scatter_rows=100), "some"),
    "c1": lambda rng: (W.config("c1").A, "all"),
    "c3_20": lambda rng: (W.config("c3", N=20).A, "all"),
    "c4_9": lambda rng: (W.config("c4", N=9).A, "all"),
    "c5_7": lambda rng: (W.config("c5", N=7).A, "all"),
    "empty_rows": lambda rng: (_banded(97, [-2, 0, 5], 0.9, rng), "all"),
}


@pytest.mark.parametrize("want_diag", [True, False])
@pytest.mark.parametrize("name", sorted(CASES))
def test_sell_plan_decodes_to_the_csr(name, want_diag):
    A, expect = CASES[name](np.random.default_rng(7))
    n, ns = A.n_rows, (A.n_rows + 31) // 32
    S = P.igs_plan_sell(n, A.rowptr, A.colind, A.values, want_diag)
    assert S is not None
    # layout invariants
    assert S["ptr"][0] == 0 and np.all(np.diff(S["ptr"]) >= 0) and np.all(S["ptr"] % 32 == 0)
    assert S["cptr"][0] == 0 and np.all(np.diff(S["cptr"]) >= 0)
    assert S["val"].size == S["ptr"][-1] and S["col"].size == S["cptr"][-1]
    assert np.array_equal(S["len"][:n], np.diff(A.rowptr).astype(np.uint8))
    assert not S["len"][n:].any() and not S["mask"][n:].any()
    diag_slice = np.diff(S["cptr"]) == 0
    width = np.diff(S["ptr"]) // 32
    for s in range(ns):
        rows = slice(32 * s, min(n, 32 * s + 32))
        if diag_slice[s]:
            lst = S["diag"][8 * s: 8 * s + width[s]]
            assert np.all(np.diff(lst) > 0)                              # ascending, distinct
            used = np.bitwise_or.reduce(S["mask"][rows]) if width[s] else 0
            assert used == (1 << width[s]) - 1                           # every listed offset is used
        else:
            assert width[s] == S["len"][rows].max() and width[s] == (S["cptr"][s + 1] - S["cptr"][s]) // 32
    nd = S["n_diag"]
    if not want_diag:                                  # nothing classified; a slice that stores
        assert nd == 0 and not width[diag_slice].any()  # no columns then stores nothing at all
    else:
        assert nd == int(diag_slice.sum())
    if not want_diag:
        pass
    elif expect == "all":
        assert nd == ns
    elif expect == "ends":
        assert 0 < nd <= 2 * (90 // 32 + 1)
    else:
        assert 0 < nd < ns
    # the arrays decode to the CSR, entry for entry, in order
    dec = _decode(n, S)
    for r in range(n):
        q0, q1 = A.rowptr[r], A.rowptr[r + 1]
        assert dec[r][0] == [int(c) for c in A.colind[q0:q1]], r
        assert np.array_equal(np.array(dec[r][1]), A.values[q0:q1]), r
    # and multiply like the oracle's row loop, bit for bit (separate multiply and add, in order)
    x = np.random.default_rng(11).standard_normal(n)
    y = np.zeros(n)
    for r in range(n):
        acc = 0.0
        for c, v in zip(*dec[r]):
            acc = acc + v * x[c]
        y[r] = acc
    assert y.tobytes() == oracle.spmv(A, x).tobytes()


def test_sell_plan_padding_is_zero_and_unreferenced():
    """Stored by list position, a row that lacks an offset keeps a zero there: the kernels
    rely on 'absent position = never read' (mask bit clear), the test on the zero."""
    A, _ = CASES["band7_masked"](np.random.default_rng(7))
    S = P.igs_plan_sell(A.n_rows, A.rowptr, A.colind, A.values, True)
    ref = np.ones(S["val"].size, bool)
    for r in range(A.n_rows):
        s, l = r >> 5, r & 31
        for j in range(8):
            if (S["mask"][r] >> j) & 1:
                ref[S["ptr"][s] + 32 * j + l] = False
    assert not S["val"][ref].any()
    assert int((~ref).sum()) == A.rowptr[-1]


def test_sell_plan_boundary_rows_and_long_rows():
    rng = np.random.default_rng(3)
    A = _banded(200, [-3, 0, 3], 0.0, rng)
    bnd = np.arange(0, 200, 7)
    S = P.igs_plan_sell(200, A.rowptr, A.colind, A.values, True, bnd)
    assert np.all(S["len"][bnd] == 255) and not S["mask"][bnd].any()
    keep = np.setdiff1d(np.arange(200), bnd)
    assert np.array_equal(S["len"][keep], np.diff(A.rowptr)[keep].astype(np.uint8))
    dec = _decode(200, S)
    assert all(dec[r] is None for r in bnd)
    assert all(dec[r][0] == [int(c) for c in A.colind[A.rowptr[r]:A.rowptr[r + 1]]] for r in keep)
    assert S["n_diag"] == 7                                      # boundary rows do not break a slice
    # a row with >= 255 entries: no SELL copy
    n = 300
    rowptr = np.arange(n + 1, dtype=np.int64)
    rowptr[1:] += 254
    colind = np.concatenate([np.arange(255), np.arange(1, n)]).astype(np.int64)
    assert P.igs_plan_sell(n, rowptr, colind, np.ones(colind.size)) is None
    with pytest.raises(P.IgsError):                              # bnd_rows must ascend
        P.igs_plan_sell(200, A.rowptr, A.colind, A.values, True, np.array([5, 3]))
