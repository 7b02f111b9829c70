"""Parity of the CUDA path (through the C-ABI) with the reference.

* every golden run of the unmodified reference (tests/golden/) -- bit-exact C
  (row_ptr, col, value bits), identical counters, identical errors;
* larger seeded inputs against the pinned CPU oracle, bit-exact, across
  SystemParams that force every category and every device kernel
  (warp / CTA / heavy-window rows, multi-batch windows, >1024-k rows).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle  # noqa: E402
from paper_2501_07056_b200 import (AccumThresholds, ContractViolation, CsrMatrix, InputError,  # noqa: E402
                                   OverBudgetError, SystemParams, compute_chunk_plan, generate, spgemm_magnus)
from paper_2501_07056_b200.planner import NUMERIC, SYMBOLIC  # noqa: E402

from golden_util import expected, inputs, runs, system  # noqa: E402

pytestmark = pytest.mark.gpu

RUNS = runs()
B200 = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 31)
HOST2M = SystemParams(cache_line_bytes=64, l2_bytes=2 << 20, memory_budget_bytes=1 << 31)
FINE4K = SystemParams(cache_line_bytes=64, l2_bytes=4096)
COARSE = SystemParams(cache_line_bytes=64, l2_bytes=1400)


def assert_same(res, ref):
    np.testing.assert_array_equal(np.asarray(res.C.row_ptr), ref.row_ptr)
    np.testing.assert_array_equal(np.asarray(res.C.col), ref.col)
    np.testing.assert_array_equal(np.asarray(res.C.val).view(np.uint64), ref.val.view(np.uint64))
    assert res.counters == ref.counters


@pytest.mark.parametrize("rec", RUNS, ids=[f"{r['case']}-{r['sys']}-{int(r.get('force_fine_only', 0))}" for r in RUNS])
def test_reference_golden(rec):
    A, B = inputs(rec["case"])
    sysp = system(rec["sys"], rec)
    if rec.get("error"):
        with pytest.raises(OverBudgetError):
            spgemm_magnus(A, B, sys=sysp, force_fine_only=rec.get("force_fine_only", False))
        return
    res = spgemm_magnus(A, B, sys=sysp, force_fine_only=rec["force_fine_only"])
    rp, col, val = expected(rec)
    np.testing.assert_array_equal(res.C.row_ptr, rp)
    np.testing.assert_array_equal(res.C.col, col)
    np.testing.assert_array_equal(res.C.val.view(np.uint64), val.view(np.uint64))
    assert res.counters == rec["counters"]


def _hub_matrix(n=4096, heavy_rows=6, heavy_deg=3000, seed=9):
    """R-MAT body plus a few rows with > 1024 nonzeros and dense hub B rows:
    exercises the global-cursor path, multi-batch windows and narrowing."""
    R = generate.rmat(12, 16, seed=seed)
    rng = np.random.default_rng(seed)
    rows = []
    rp = np.asarray(R.row_ptr)
    for i in range(n):
        r = np.asarray(R.col[rp[i]:rp[i + 1]], dtype=np.int64)
        if i < heavy_rows:
            r = np.union1d(r, rng.choice(n, size=heavy_deg, replace=False))
        if 10 <= i < 14:  # dense-ish hub rows of B
            r = np.union1d(r, np.arange(0, n, 2))
        rows.append(r)
    rp2 = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=rp2[1:])
    col = np.concatenate(rows).astype(np.int32)
    val = generate.uniform_pm1(seed, 0xAB, np.arange(col.size, dtype=np.uint64))
    return CsrMatrix(n, n, rp2, col, val)


CASES = {
    "rmat14": lambda: (generate.rmat(14, 16, seed=31),) * 2,
    "hub": lambda: (_hub_matrix(),) * 2,
    "uniform": lambda: (generate.uniform_rows(8192, 8192, 16, seed=1),) * 2,
    "stencil": lambda: (generate.stencil27(20),) * 2,
    "AB": lambda: (generate.uniform_rows(4096, 1 << 16, 8, seed=2), generate.uniform_rows(1 << 16, 1 << 20, 8, seed=3)),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("sysname", ["b200", "host2m", "fine4k", "coarse"])
def test_against_oracle(case, sysname):
    A, B = CASES[case]()
    sysp = {"b200": B200, "host2m": HOST2M, "fine4k": FINE4K, "coarse": COARSE}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    res = spgemm_magnus(A, B, sys=sysp)
    assert_same(res, ref)


def test_force_fine_only_and_thresholds():
    A = generate.rmat(13, 16, seed=4)
    ref = oracle.spgemm(A, A, COARSE, force_fine_only=True)
    assert_same(spgemm_magnus(A, A, sys=COARSE, force_fine_only=True), ref)
    th = AccumThresholds(sort_dense_crossover=64, sort_sweet_spot=8)
    ref = oracle.spgemm(A, A, FINE4K, thresholds=th)
    assert_same(spgemm_magnus(A, A, sys=FINE4K, thresholds=th), ref)


def test_device_tensors_int32_row_ptr_and_determinism():
    A = generate.rmat(13, 16, seed=5)
    dev = torch.device("cuda")
    Ad = CsrMatrix(A.n_rows, A.n_cols, torch.from_numpy(A.row_ptr.astype(np.int32)).to(dev),
                   torch.from_numpy(A.col).to(dev), torch.from_numpy(A.val).to(dev))
    r1 = spgemm_magnus(Ad, Ad, sys=B200)
    r2 = spgemm_magnus(Ad, Ad, sys=B200)
    assert r1.C.col.is_cuda
    assert torch.equal(r1.C.row_ptr, r2.C.row_ptr) and torch.equal(r1.C.col, r2.C.col)
    assert torch.equal(r1.C.val.view(torch.int64), r2.C.val.view(torch.int64))
    ref = oracle.spgemm(A, A, B200)
    np.testing.assert_array_equal(r1.C.row_ptr.cpu().numpy(), ref.row_ptr)
    np.testing.assert_array_equal(r1.C.val.cpu().numpy().view(np.uint64), ref.val.view(np.uint64))


def test_edge_shapes():
    E = CsrMatrix(3, 5, np.zeros(4, np.int64), np.empty(0, np.int32), np.empty(0))
    F = generate.uniform_rows(5, 7, 3, seed=1)
    r = spgemm_magnus(E, F, sys=B200)
    assert r.C.nnz == 0 and list(r.C.row_ptr) == [0, 0, 0, 0]
    Z = CsrMatrix(0, 5, np.zeros(1, np.int64), np.empty(0, np.int32), np.empty(0))
    r = spgemm_magnus(Z, F, sys=B200)
    assert r.C.n_rows == 0 and r.C.nnz == 0
    with pytest.raises(InputError):
        spgemm_magnus(F, F, sys=B200)   # 5x7 . 5x7: dimension mismatch


@pytest.mark.parametrize("crossover", [512, 1024, 3000])
def test_heavy_paths_by_crossover(crossover):
    """crossover <= 512 runs the binned heavy path, above it the windowed heavy kernel."""
    th = AccumThresholds(sort_dense_crossover=crossover, sort_sweet_spot=8)
    for A, B in (CASES["hub"](), CASES["rmat14"]()):
        for sysp in (B200, FINE4K):
            ref = oracle.spgemm(A, B, sysp, thresholds=th)
            assert_same(spgemm_magnus(A, B, sys=sysp, thresholds=th), ref)


def _hot_chunk_matrix(seed=11):
    """Rows whose products pile into single chunks (2^20 columns): one row with ~220K
    products inside columns [0, 4096) -- more than one big-chunk reducer part --, rows
    with mid-size hot chunks, and light rows."""
    rng = np.random.default_rng(seed)
    m, n = 1 << 12, 1 << 20
    rows = []
    for i in range(m):
        if i == 0:
            r = np.arange(1, 1 + 220)                        # 220 k's ...
        elif i < 40:
            r = rng.choice(20000, size=int(rng.integers(20, 200)), replace=False)
        else:
            r = rng.choice(20000, size=int(rng.integers(1, 9)), replace=False)
        rows.append(np.unique(r))
    B_rows = []
    for k in range(20000):                                  # rows >= 20000 of B are empty
        if 1 <= k <= 220:                                   # ... each B row dense in columns [0, 4096)
            B_rows.append(rng.choice(4096, size=1000, replace=False))
        elif k < 2000:
            B_rows.append(rng.choice(1 << 15, size=int(rng.integers(50, 400)), replace=False))
        else:
            B_rows.append(rng.choice(n, size=int(rng.integers(1, 16)), replace=False))

    def csr(rr, nrows, nc, seedv):
        rr = [np.unique(r) for r in rr]
        rp = np.zeros(nrows + 1, np.int64)
        np.cumsum([len(r) for r in rr], out=rp[1:len(rr) + 1])
        rp[len(rr) + 1:] = rp[len(rr)]
        col = np.concatenate(rr).astype(np.int32)
        val = generate.uniform_pm1(seedv, 0xCD, np.arange(col.size, dtype=np.uint64))
        return CsrMatrix(nrows, nc, rp, col, val)

    return csr(rows, m, n, seed), csr(B_rows, n, n, seed + 1)


@pytest.mark.parametrize("sysname", ["b200", "fine4k"])
def test_hot_chunks_against_oracle(sysname):
    A, B = _hot_chunk_matrix()
    sysp = {"b200": B200, "fine4k": FINE4K}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)


def test_heavy_rows_1024_column_chunks():
    """R-MAT 2^15 under the B200 parameters: numeric chunks of 1024 columns (32 bitmap
    words), where the big-chunk reducer marks its own column bitmaps."""
    A = generate.rmat(15, 16, seed=7)
    ref = oracle.spgemm(A, A, B200)
    assert_same(spgemm_magnus(A, A, sys=B200), ref)


@pytest.mark.parametrize("case", ["rmat14", "hub", "hot", "rmat15"])
@pytest.mark.parametrize("sysname", ["b200", "fine4k"])
def test_direct_heavy_path(case, sysname, monkeypatch):
    """The direct heavy path (MAGNUS_HEAVY_PATH=direct, no reorder buffer) gives the same
    bits as the reference association."""
    monkeypatch.setenv("MAGNUS_HEAVY_PATH", "direct")
    if case == "hot":
        A, B = _hot_chunk_matrix()
    elif case == "rmat15":
        A = B = generate.rmat(15, 16, seed=7)
    else:
        A, B = CASES[case]()
    sysp = {"b200": B200, "fine4k": FINE4K}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)


@pytest.mark.parametrize("batch_elems", [0, 20000])
def test_numeric_host_readback(batch_elems, monkeypatch):
    """magnus_numeric_host: C read back into host buffers (overlapped with later heavy-row
    batches; MAGNUS_BATCH_ELEMS forces many batches) equals C on the device, and the
    heavy-row batches (in row order) give the oracle's bits."""
    from paper_2501_07056_b200 import MagnusPlan
    if batch_elems:
        monkeypatch.setenv("MAGNUS_BATCH_ELEMS", str(batch_elems))
    A = generate.rmat(14, 16, seed=31)
    dev = torch.device("cuda")
    Ad = CsrMatrix(A.n_rows, A.n_cols, torch.from_numpy(A.row_ptr).to(dev), torch.from_numpy(A.col).to(dev),
                   torch.from_numpy(A.val).to(dev))
    plan = MagnusPlan(Ad, Ad, sys=B200)
    rp = plan.symbolic()
    hc = torch.empty(plan.nnz, dtype=torch.int32).pin_memory()
    hv = torch.empty(plan.nnz, dtype=torch.float64).pin_memory()
    C, _ = plan.numeric(rp, host_out=(hc, hv))
    plan.close()
    assert torch.equal(hc, C.col.cpu()) and torch.equal(hv.view(torch.int64), C.val.cpu().view(torch.int64))
    ref = oracle.spgemm(A, A, B200)
    np.testing.assert_array_equal(rp.cpu().numpy(), ref.row_ptr)
    np.testing.assert_array_equal(hc.numpy().view(np.uint32), ref.col)
    np.testing.assert_array_equal(hv.numpy().view(np.uint64), ref.val.view(np.uint64))


def _broken(kind):
    A = generate.rmat(10, 8, seed=12)
    rp = np.asarray(A.row_ptr, np.int64).copy()
    col = np.asarray(A.col).astype(np.uint32).copy()
    val = np.asarray(A.val).copy()
    row = int(np.argmax(np.diff(rp) >= 3))
    if kind == "b_col_range":
        col[rp[row]] = A.n_cols + 5
    elif kind == "dup":
        col[rp[row] + 1] = col[rp[row]]
    elif kind == "unsorted":
        col[rp[row]], col[rp[row] + 1] = col[rp[row] + 1], col[rp[row]]
    elif kind == "row_ptr":
        rp[3] = rp[4] + 2
    return A, CsrMatrix(A.n_rows, A.n_cols, rp, col, val)


@pytest.mark.parametrize("kind,exc", [("b_col_range", ContractViolation), ("dup", InputError),
                                      ("unsorted", InputError), ("row_ptr", InputError)])
def test_input_contract_errors(kind, exc):
    """Out-of-span B columns -> ContractViolation (magnus.py:208-209, 245-246); malformed row_ptr
    and non-canonical rows -> InputError (validate_csr, matrix.py:119-150), checked on the device
    before any kernel indexes through the inputs."""
    A, bad = _broken(kind)
    with pytest.raises(exc):
        spgemm_magnus(A, bad, sys=B200)
    if kind != "b_col_range":
        with pytest.raises(InputError):
            spgemm_magnus(bad, A, sys=B200)
    # A column outside B's rows
    A2 = generate.rmat(10, 8, seed=12)
    col = np.asarray(A2.col).astype(np.uint32).copy()
    col[7] = A2.n_cols + 1
    with pytest.raises(InputError):
        spgemm_magnus(CsrMatrix(A2.n_rows, A2.n_cols, A2.row_ptr, col, A2.val), A2, sys=B200)
    # the library still works afterwards
    assert spgemm_magnus(A, A, sys=B200).C.nnz > 0


@pytest.mark.parametrize("sysname", ["b200", "coarse"])
def test_phase_entry_points(sysname):
    """magnus_symbolic / magnus_numeric / categorize_rows with the reference signatures
    (magnus.py:68, 420, 459) give the full pipeline's result."""
    from paper_2501_07056_b200 import categorize_rows, magnus_numeric, magnus_symbolic, row_intermediate_stats
    sysp = {"b200": B200, "coarse": COARSE}[sysname]
    A = generate.rmat(12, 16, seed=21)
    th = AccumThresholds()
    plan_s = compute_chunk_plan(sysp, A.n_cols, SYMBOLIC)
    plan_n = compute_chunk_plan(sysp, A.n_cols, NUMERIC)
    st = row_intermediate_stats(A, A)
    cats = categorize_rows(st, plan_s, sysp, th)
    ref = oracle.spgemm(A, A, sysp)
    counts = cats.counts
    assert [counts[k] for k in ("sort", "dense", "fine", "coarse")] == [ref.counters[k] for k in
                                                                        ("rows_sort", "rows_dense", "rows_fine",
                                                                         "rows_coarse")]
    rp = magnus_symbolic(A, A, plan_s, cats, st, sysp, th)
    np.testing.assert_array_equal(rp, ref.row_ptr)
    res = magnus_numeric(A, A, rp, plan_n, cats, st, sysp, th)
    assert_same(res, ref)
    # a row_ptr from elsewhere is re-derived and checked; a wrong one is a ContractViolation
    res2 = magnus_numeric(A, A, rp.copy(), plan_n, cats, st, sysp, th)
    np.testing.assert_array_equal(res2.C.val.view(np.uint64), ref.val.view(np.uint64))
    bad = rp.copy()
    bad[5:] += 1
    with pytest.raises(ContractViolation):
        magnus_numeric(A, A, bad, plan_n, cats, st, sysp, th)


def test_workspace_pool_release():
    from paper_2501_07056_b200 import _lib
    A = generate.rmat(13, 16, seed=2)
    spgemm_magnus(A, A, sys=B200)
    assert _lib.workspace_reserved() > 0
    _lib.release_workspace()
    assert _lib.workspace_reserved() == 0
    assert spgemm_magnus(A, A, sys=B200).C.nnz > 0


@pytest.mark.parametrize("case", ["rmat14", "hub", "hot", "rmat15"])
@pytest.mark.parametrize("sysname", ["b200", "fine4k"])
@pytest.mark.parametrize("path", ["direct", "fused"])
def test_direct_big_chunk_path(case, sysname, path, monkeypatch):
    """Big chunks straight from B (MAGNUS_BIG_PATH=direct, big_direct.cuh, or =fused, fused_big.cuh:
    no reorder buffer for them; the small chunks' buffer holds small-chunk products only) give the
    reference's bits."""
    monkeypatch.setenv("MAGNUS_BIG_PATH", path)
    if case == "hot":
        A, B = _hot_chunk_matrix()
    elif case == "rmat15":
        A = B = generate.rmat(15, 16, seed=7)
    else:
        A, B = CASES[case]()
    sysp = {"b200": B200, "fine4k": FINE4K}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)
    monkeypatch.setenv("MAGNUS_BATCH_ELEMS", "20000")   # many small-chunk batches
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)


def test_caller_owned_workspace():
    """magnus_workspace_bytes / magnus_set_workspace: the reorder buffer in caller
    memory -- at the minimum size (many batches) and at the preferred one -- gives the same bits."""
    from paper_2501_07056_b200 import MagnusPlan
    A = generate.rmat(14, 16, seed=31)
    ref = oracle.spgemm(A, A, B200)
    dev = torch.device("cuda")
    Ad = CsrMatrix(A.n_rows, A.n_cols, torch.from_numpy(A.row_ptr).to(dev), torch.from_numpy(A.col).to(dev),
                   torch.from_numpy(A.val).to(dev))
    for which in (1, 0):
        plan = MagnusPlan(Ad, Ad, sys=B200)
        rp = plan.symbolic()
        pref, mini = plan.workspace_bytes()
        assert 0 < mini <= pref
        ws = torch.empty((pref, mini)[which], dtype=torch.uint8, device=dev)
        C, _ = plan.numeric(rp, workspace=ws)
        plan.close()
        np.testing.assert_array_equal(C.col.cpu().numpy().view(np.uint32), ref.col)
        np.testing.assert_array_equal(C.val.cpu().numpy().view(np.uint64), ref.val.view(np.uint64))
    plan = MagnusPlan(Ad, Ad, sys=B200)
    rp = plan.symbolic()
    with pytest.raises(InputError):
        plan.numeric(rp, workspace=torch.empty(16, dtype=torch.uint8, device=dev))
    plan.close()


COARSE16K = SystemParams(cache_line_bytes=64, l2_bytes=6000)   # m_max 2^16: several coarse chunks for 2^20 columns


@pytest.mark.parametrize("case", ["rmat14", "hub", "rmat15", "AB"])
@pytest.mark.parametrize("sysname", ["coarse", "coarse16k"])
def test_device_coarse_level(case, sysname, monkeypatch):
    """Coarse-category rows go through the device coarse level (coarse_rows.cuh: CSC view of the
    batch's A rows, every referenced B row staged once, row-linked (row, coarse chunk) buckets, fine
    level per bucket -- reference magnus.py:317-406) and give the reference's bits; so does the
    fine-level expand (MAGNUS_COARSE_PATH=fine), and several device batches."""
    from paper_2501_07056_b200 import MagnusPlan
    if case == "rmat15":
        A = B = generate.rmat(15, 16, seed=7)
    else:
        A, B = CASES[case]()
    sysp = {"coarse": COARSE, "coarse16k": COARSE16K}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    plan = MagnusPlan(A, B, sys=sysp)
    rp = plan.symbolic()
    res, _counters = plan.numeric(rp)
    st = plan.ctx.coarse_level_stats()
    to_np = lambda t: t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)   # noqa: E731
    np.testing.assert_array_equal(to_np(res.row_ptr), ref.row_ptr)
    np.testing.assert_array_equal(to_np(res.col).astype(np.int64) & 0xFFFFFFFF, ref.col.astype(np.int64))
    np.testing.assert_array_equal(to_np(res.val).view(np.uint64), ref.val.view(np.uint64))
    if ref.counters["rows_coarse"] > 0 and case != "AB":
        assert st["rows"] > 0 and st["batches"] >= 1, st   # the coarse level really ran
    plan.close()
    monkeypatch.setenv("MAGNUS_BATCH_ELEMS", "300000")   # several heavy-row batches -> several coarse batches
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)
    monkeypatch.setenv("MAGNUS_COARSE_PATH", "fine")
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)


@pytest.mark.parametrize("knob", ["MAGNUS_SERIAL=0", "MAGNUS_LIGHT_SIDE=0", "MAGNUS_FUSED_ROWS=0",
                                  "MAGNUS_HEAVY_SYMBOLIC=window", "MAGNUS_BATCH_FRAC=0.05"])
def test_device_path_knobs_do_not_change_results(knob, monkeypatch):
    """The tuning knobs of the device path (pipelined reducers on side streams, light rows on
    the main stream, unfused warp rows, the windowed heavy symbolic kernel, a small reorder buffer) only change
    the execution strategy: the reference's bits come out under each of them, also with many heavy-row batches."""
    name, value = knob.split("=")
    A = generate.rmat(14, 16, seed=31)
    ref = oracle.spgemm(A, A, B200)
    monkeypatch.setenv(name, value)
    assert_same(spgemm_magnus(A, A, sys=B200), ref)
    monkeypatch.setenv("MAGNUS_BATCH_ELEMS", "150000")
    assert_same(spgemm_magnus(A, A, sys=B200), ref)
    H = _hub_matrix()
    assert_same(spgemm_magnus(H, H, sys=FINE4K), oracle.spgemm(H, H, FINE4K))


def _wide_matrix(n_rows, n_cols_b, per_row, seed):
    rng = np.random.default_rng(seed)
    cols = np.sort(rng.choice(np.arange(0, n_cols_b, max(1, n_cols_b // 50000), dtype=np.int64), size=(n_rows, per_row)), axis=1)
    for r in range(n_rows):   # distinct, ascending per row
        while np.unique(cols[r]).size < per_row:
            cols[r] = np.sort(rng.choice(np.arange(0, n_cols_b, max(1, n_cols_b // 50000), dtype=np.int64), size=per_row))
    rp = np.arange(n_rows + 1, dtype=np.int64) * per_row
    val = generate.uniform_pm1(seed, 0xCD, np.arange(n_rows * per_row, dtype=np.uint64))
    return CsrMatrix(n_rows, n_cols_b, rp, cols.reshape(-1).astype(np.uint32), val)


@pytest.mark.parametrize("n_cols", [(1 << 32) - 3, (1 << 31) + 11, 1 << 26])
def test_wide_column_space(n_cols):
    """Columns up to 2^32 - 4 (uint32 indices with the top bit set): light rows with 64-bit sort keys and a heavy
    row (2000 nonzeros of A) on whichever heavy path the plan allows -- the reference's bits."""
    rng = np.random.default_rng(5)
    nk = 2000
    B = _wide_matrix(nk, n_cols, 12, seed=11)
    rows = [np.sort(rng.choice(nk, size=(nk if i == 0 else 5), replace=False)) for i in range(64)]
    rp = np.zeros(65, np.int64)
    np.cumsum([len(r) for r in rows], out=rp[1:])
    col = np.concatenate(rows).astype(np.int32)
    A = CsrMatrix(64, nk, rp, col, generate.uniform_pm1(3, 0xEE, np.arange(col.size, dtype=np.uint64)))
    for sysp in (B200, HOST2M):
        ref = oracle.spgemm(A, B, sysp)
        assert_same(spgemm_magnus(A, B, sys=sysp), ref)


@pytest.mark.parametrize("sysname", ["b200", "fine4k", "coarse"])
def test_signed_zeros_and_cancellation(sysname):
    """Cancellation (pairs of identical B rows with opposite A coefficients: every sum is zero or a rounding residue
    that depends on the association), explicit +0.0 / -0.0 values in A and B: the structural entries stay, and every
    residue and the sign of every zero are the reference's -- on warp, CTA and heavy rows."""
    rng = np.random.default_rng(17)
    n, nk = 96, 1500
    base = generate.uniform_rows(nk // 2, 1 << 15, 24, seed=9)
    # B: every row twice (k and k + nk/2 are identical), a tenth of the values +-0.0
    rpb = np.concatenate([np.asarray(base.row_ptr), np.asarray(base.row_ptr)[1:] + int(base.row_ptr[-1])])
    colb = np.concatenate([np.asarray(base.col), np.asarray(base.col)])
    valb = np.concatenate([np.asarray(base.val), np.asarray(base.val)]).copy()
    z = rng.random(valb.size) < 0.1
    valb[z] = np.where(rng.random(int(z.sum())) < 0.5, 0.0, -0.0)
    valb[valb.size // 2:] = valb[:valb.size // 2]
    B = CsrMatrix(nk, 1 << 15, rpb.astype(np.int64), colb.astype(np.int32), valb)
    rows, vals = [], []
    for i in range(n):
        m = (700, 60, 8)[i % 3] if i else 740   # heavy, CTA and warp rows
        ks = np.sort(rng.choice(nk // 2, size=m, replace=False))
        a = generate.uniform_pm1(i + 1, 0xAA, np.arange(m, dtype=np.uint64))
        a[rng.random(m) < 0.05] = -0.0
        rows.append(np.concatenate([ks, ks + nk // 2]))      # k and its twin ...
        vals.append(np.concatenate([a, -a]))                 # ... with opposite coefficients
    rp = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=rp[1:])
    A = CsrMatrix(n, nk, rp, np.concatenate(rows).astype(np.int32), np.concatenate(vals))
    sysp = {"b200": B200, "fine4k": FINE4K, "coarse": COARSE}[sysname]
    ref = oracle.spgemm(A, B, sysp)
    assert ref.val.size and np.mean(np.abs(ref.val) < 1e-12) > 0.99   # (near-)exact cancellation everywhere
    assert_same(spgemm_magnus(A, B, sys=sysp), ref)
