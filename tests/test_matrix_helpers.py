"""Host-side CSR helpers with the reference's API (matrix.py:47-224): validate_csr reports,
csr_from_arrays / csr_from_triplets, canonicalize_csr, csr_rows_to_csc; and the pure
categorize_rows rule (magnus.py:68-94).  Checked against the unmodified reference when it is
importable (this container), and by properties everywhere."""

import os
import sys

import numpy as np
import pytest

from paper_2501_07056_b200 import (AccumThresholds, CsrMatrix, RowStats, SystemParams, canonicalize_csr,
                                   compute_chunk_plan, csr_from_arrays, csr_from_triplets, csr_rows_to_csc, generate,
                                   validate_csr)
from paper_2501_07056_b200.planner import SYMBOLIC

REF = "/root/reference/pkg/src"


def _ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (only in the build container)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import spgemm.magnus as rm
    import spgemm.matrix as rmat
    return rmat, rm


def _bad_matrices():
    A = generate.rmat(8, 8, seed=3)
    rp = np.asarray(A.row_ptr, np.int64)
    out = {"ok": A}
    out["short_rp"] = CsrMatrix(A.n_rows, A.n_cols, rp[:-1], A.col, A.val)
    r = rp.copy(); r[0] = 1
    out["rp0"] = CsrMatrix(A.n_rows, A.n_cols, r, A.col, A.val)
    r = rp.copy(); r[5] = r[6] + 1
    out["decreasing"] = CsrMatrix(A.n_rows, A.n_cols, r, A.col, A.val)
    out["lengths"] = CsrMatrix(A.n_rows, A.n_cols, rp, A.col[:-1], A.val)
    c = np.asarray(A.col).astype(np.uint32).copy(); c[17] = A.n_cols + 3
    out["range"] = CsrMatrix(A.n_rows, A.n_cols, rp, c, A.val)
    c = np.asarray(A.col).astype(np.uint32).copy()
    row = int(np.argmax(np.diff(rp) >= 3))
    c[rp[row] + 1] = c[rp[row]]
    out["dup"] = CsrMatrix(A.n_rows, A.n_cols, rp, c, A.val)
    out["dup_noncanonical"] = CsrMatrix(A.n_rows, A.n_cols, rp, c, A.val, canonical=False)
    return out


def test_validate_csr_reports():
    ms = _bad_matrices()
    assert validate_csr(ms["ok"]) and validate_csr(ms["dup_noncanonical"])
    for k in ("short_rp", "rp0", "decreasing", "lengths", "range", "dup"):
        rep = validate_csr(ms[k])
        assert not rep and rep.message != "OK", k


def test_validate_csr_matches_reference():
    rmat, _ = _ref()
    for k, m in _bad_matrices().items():
        rm = rmat.CsrMatrix(m.n_rows, m.n_cols, np.asarray(m.row_ptr, np.int64), np.asarray(m.col).astype(np.uint32),
                            np.asarray(m.val), m.canonical)
        try:
            b = rmat.validate_csr(rm)
        except IndexError:   # the reference's own check indexes past the end for trailing empty rows
            continue
        a = validate_csr(m)
        assert (bool(a), a.message, a.index) == (bool(b), b.message, b.index), k


def test_csr_from_arrays_and_triplets():
    rng = np.random.default_rng(4)
    r = rng.integers(0, 50, 400)
    c = rng.integers(0, 70, 400)
    v = rng.standard_normal(400)
    m = csr_from_arrays(r, c, v, 50, 70)
    assert validate_csr(m)
    np.testing.assert_allclose(m.to_dense(), _dense(r, c, v, 50, 70))
    t = csr_from_triplets(zip(r.tolist(), c.tolist(), v.tolist()), 50, 70)
    np.testing.assert_array_equal(t.col, m.col)
    np.testing.assert_array_equal(t.val.view(np.uint64), m.val.view(np.uint64))
    e = csr_from_triplets([], 3, 4)
    assert e.nnz == 0 and e.row_ptr.tolist() == [0, 0, 0, 0]


def _dense(r, c, v, n, m):
    d = np.zeros((n, m))
    np.add.at(d, (r, c), v)
    return d


def test_csr_from_arrays_matches_reference():
    rmat, _ = _ref()
    rng = np.random.default_rng(5)
    r = rng.integers(0, 64, 3000)
    c = rng.integers(0, 1000, 3000)
    v = rng.uniform(-1, 1, 3000)
    a, b = csr_from_arrays(r, c, v, 64, 1000), rmat.csr_from_arrays(r, c, v, 64, 1000)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col, b.col)
    assert a.col.dtype == b.col.dtype
    np.testing.assert_array_equal(a.val.view(np.uint64), b.val.view(np.uint64))


def test_canonicalize_and_csc_match_reference():
    rmat, _ = _ref()
    A = generate.rmat(9, 8, seed=6)
    rp = np.asarray(A.row_ptr, np.int64)
    rng = np.random.default_rng(7)
    perm = np.concatenate([rp[i] + rng.permutation(rp[i + 1] - rp[i]) for i in range(A.n_rows)])
    col = np.asarray(A.col).astype(np.uint32)[perm]
    val = np.asarray(A.val)[perm]
    mine = canonicalize_csr(CsrMatrix(A.n_rows, A.n_cols, rp.copy(), col.copy(), val.copy(), canonical=False))
    ref = rmat.canonicalize_csr(rmat.CsrMatrix(A.n_rows, A.n_cols, rp.copy(), col.copy(), val.copy(), False))
    assert mine.canonical and ref.canonical
    np.testing.assert_array_equal(mine.col, ref.col)
    np.testing.assert_array_equal(mine.val.view(np.uint64), ref.val.view(np.uint64))
    rows = np.sort(rng.choice(A.n_rows, 60, replace=False))
    a = csr_rows_to_csc(A, rows)
    b = rmat.csr_rows_to_csc(rmat.CsrMatrix(A.n_rows, A.n_cols, rp, np.asarray(A.col).astype(np.uint32),
                                            np.asarray(A.val)), rows)
    np.testing.assert_array_equal(a.col_ptr, b.col_ptr)
    np.testing.assert_array_equal(a.row, b.row)
    np.testing.assert_array_equal(a.val.view(np.uint64), b.val.view(np.uint64))
    assert a.nnz == b.nnz


def test_csr_rows_to_csc_properties():
    A = generate.rmat(8, 8, seed=2)
    rows = np.array([1, 5, 9, 40, 41, 200])
    csc = csr_rows_to_csc(A, rows)
    d = A.to_dense()[rows]
    back = np.zeros_like(d)
    for j in range(A.n_cols):
        for q in range(csc.col_ptr[j], csc.col_ptr[j + 1]):
            back[csc.row[q], j] += csc.val[q]
        seg = csc.row[csc.col_ptr[j]:csc.col_ptr[j + 1]]
        assert (np.diff(seg) > 0).all()
    np.testing.assert_array_equal(back, d)
    with pytest.raises(Exception):
        csr_rows_to_csc(A, np.array([3, 2]))


@pytest.mark.parametrize("use_coarse_l2", [2 << 20, 1400])
def test_categorize_rows_matches_reference(use_coarse_l2):
    _, rm = _ref()
    import spgemm.gustavson as rg
    import spgemm.planner as rp_
    from paper_2501_07056_b200.magnus import categorize_rows
    A = generate.rmat(11, 16, seed=8)
    sysp = SystemParams(cache_line_bytes=64, l2_bytes=use_coarse_l2)
    th = AccumThresholds()
    RA = rm.CsrMatrix(A.n_rows, A.n_cols, np.asarray(A.row_ptr, np.int64), np.asarray(A.col).astype(np.uint32),
                      np.asarray(A.val))
    st = rg.row_intermediate_stats(RA, RA)
    rsys = rp_.SystemParams(cache_line_bytes=64, l2_bytes=use_coarse_l2)
    plan_r = rp_.compute_chunk_plan(rsys, A.n_cols, rp_.SYMBOLIC)
    ref = rm.categorize_rows(st, plan_r, rsys, rm.AccumThresholds())
    mine = categorize_rows(RowStats(st.inter_size, st.min_col, st.max_col),
                           compute_chunk_plan(sysp, A.n_cols, SYMBOLIC), sysp, th)
    for f in ("sort_rows", "dense_rows", "fine_rows", "coarse_rows"):
        np.testing.assert_array_equal(getattr(mine, f), getattr(ref, f))
