"""Parity of the device Gustavson baselines (csrc/baselines.cuh through the C-ABI
magnus_gd_* / magnus_esc_*) with the reference's gustavson_dense / gustavson_esc
(gustavson.py:155-268): bit-exact against the reference's golden runs and the pinned
oracle; batching, long rows, host and device inputs, contract errors."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import golden_util as gu  # noqa: E402
import gustavson_golden as gg  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2501_07056_b200 import (ContractViolation, CsrMatrix, generate, gustavson,  # noqa: E402
                                   gustavson_dense, gustavson_dense_numeric, gustavson_dense_symbolic,
                                   gustavson_esc, gustavson_esc_numeric, spgemm_magnus)

pytestmark = pytest.mark.gpu

FNS = {"dense": gustavson_dense, "esc": gustavson_esc}


def _np(x):
    return x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def assert_bits(res, rp, col, val):
    np.testing.assert_array_equal(_np(res.C.row_ptr), rp)
    np.testing.assert_array_equal(_np(res.C.col).view(np.uint32), col)
    np.testing.assert_array_equal(_np(res.C.val).view(np.uint64), np.asarray(val).view(np.uint64))


@pytest.mark.parametrize("case", gg.cases())
@pytest.mark.parametrize("algo", ["dense", "esc"])
def test_reference_golden(case, algo):
    A, B = gu.inputs(case)
    rp, col, val, counters = gg.expected(case, algo)
    res = FNS[algo](A, B)
    assert_bits(res, rp, col, val)
    assert res.counters == counters
    assert set(res.phase_timings) == {"setup", "symbolic", "numeric", "post"}


def _long_rows(seed=3):
    """R-MAT body plus rows whose product has > 4096 distinct columns (bitmap-scan emission)."""
    R = generate.rmat(13, 16, seed=seed)
    rng = np.random.default_rng(seed)
    rp = np.asarray(R.row_ptr).astype(np.int64)
    rows = [np.asarray(R.col[rp[i]:rp[i + 1]]) for i in range(R.n_rows)]
    for i in (0, 17, 4095):
        rows[i] = np.sort(rng.choice(R.n_cols, size=1500, replace=False)).astype(np.int32)
    nrp = np.zeros(R.n_rows + 1, np.int64)
    np.cumsum([r.size for r in rows], out=nrp[1:])
    col = np.concatenate(rows).astype(np.int32)
    return CsrMatrix(R.n_rows, R.n_cols, nrp, col, rng.uniform(-1, 1, col.size))


@pytest.mark.parametrize("algo", ["dense", "esc"])
def test_oracle_rmat_and_long_rows(algo):
    for A in (generate.rmat(12, 8, seed=4), _long_rows()):
        ref = oracle.gustavson(A, A, esc=(algo == "esc"))
        assert np.diff(ref.row_ptr).max() > 4096 or A.n_rows == 4096
        res = FNS[algo](A, A)
        assert_bits(res, ref.row_ptr, ref.col, ref.val)
        assert res.counters == ref.counters


def test_rectangular_ab_and_device_inputs():
    A = generate.uniform_rows(3000, 50000, 7, seed=5)
    B = generate.uniform_rows(50000, 70000, 5, seed=6)
    for algo in ("dense", "esc"):
        ref = oracle.gustavson(A, B, esc=(algo == "esc"))
        dA = CsrMatrix(A.n_rows, A.n_cols, torch.as_tensor(np.asarray(A.row_ptr)).cuda(),
                       torch.as_tensor(np.asarray(A.col)).cuda(), torch.as_tensor(np.asarray(A.val)).cuda())
        dB = CsrMatrix(B.n_rows, B.n_cols, torch.as_tensor(np.asarray(B.row_ptr)).cuda(),
                       torch.as_tensor(np.asarray(B.col)).cuda(), torch.as_tensor(np.asarray(B.val)).cuda())
        res = FNS[algo](dA, dB)
        assert res.C.col.is_cuda
        assert_bits(res, ref.row_ptr, ref.col, ref.val)


def test_esc_batches_and_small_scratch(monkeypatch):
    A = generate.rmat(11, 8, seed=8)
    ref_e = oracle.gustavson(A, A, esc=True)
    ref_d = oracle.gustavson(A, A, esc=False)
    rp = gustavson_dense_symbolic(A, A)
    np.testing.assert_array_equal(rp, ref_e.row_ptr)
    monkeypatch.setattr(gustavson, "ESC_BATCH_PRODUCTS", 777)
    res = gustavson_esc_numeric(A, A, rp)
    assert_bits(res, ref_e.row_ptr, ref_e.col, ref_e.val)
    # one dense accumulator only: every row through the same CTA, bitmaps reused row after row
    monkeypatch.setattr(gustavson._Pair, "scratch", lambda self: torch.empty(
        int(gustavson._lib.lib().magnus_gd_scratch_bytes(self.B.n_cols, 1)) + 16, dtype=torch.uint8,
        device=self.device))
    res = gustavson_dense_numeric(A, A, rp)
    assert_bits(res, ref_d.row_ptr, ref_d.col, ref_d.val)


def test_contract_violation():
    A = generate.rmat(10, 8, seed=2)
    rp = gustavson_dense_symbolic(A, A).copy()
    bad = rp.copy()
    bad[5:] += 1
    for fn in (gustavson_dense_numeric, gustavson_esc_numeric):
        with pytest.raises(ContractViolation):
            fn(A, A, bad)
        with pytest.raises(ContractViolation):
            fn(A, A, rp[:-1])


def test_agrees_with_magnus_pattern():
    A = generate.rmat(12, 16, seed=11)
    m = spgemm_magnus(A, A)
    for fn in (gustavson_dense, gustavson_esc):
        g = fn(A, A)
        np.testing.assert_array_equal(g.C.row_ptr, m.C.row_ptr)
        np.testing.assert_array_equal(g.C.col, m.C.col)
        np.testing.assert_allclose(g.C.val, m.C.val, rtol=1e-12, atol=1e-12 * np.abs(m.C.val).max())
