"""CSR container mirroring the reference's `CsrMatrix` (matrix.py:18-44).

Same fields (``n_rows, n_cols, row_ptr, col, val, canonical``).  Arrays may be
numpy (host, the reference's own representation) or torch tensors (host or
CUDA).  ``col`` is stored as int32 where the reference uses uint32
(`util.py:47-49`): every config has fewer than 2^31 columns and torch has no
uint32 arithmetic; the C-ABI reads the same bits as uint32.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InputError


@dataclass
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_ptr: object
    col: object
    val: object
    canonical: bool = True

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def row_slice(self, i):
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return self.col[lo:hi], self.val[lo:hi]

    def numpy(self) -> "CsrMatrix":
        """Host numpy copy (no-op for numpy inputs)."""
        def cv(x):
            if isinstance(x, np.ndarray):
                return x
            return x.detach().cpu().numpy()
        return CsrMatrix(self.n_rows, self.n_cols, cv(self.row_ptr), cv(self.col), cv(self.val), self.canonical)

    def to_dense(self) -> np.ndarray:
        m = self.numpy()
        if m.n_rows * m.n_cols > 2**26:
            raise InputError("to_dense is restricted to small matrices")
        d = np.zeros((m.n_rows, m.n_cols))
        rows = np.repeat(np.arange(m.n_rows), np.diff(np.asarray(m.row_ptr, dtype=np.int64)))
        np.add.at(d, (rows, np.asarray(m.col).astype(np.int64)), m.val)
        return d


@dataclass
class RowStats:
    """Per-row intermediate-product statistics (reference matrix.py:227-239)."""

    inter_size: object
    min_col: object
    max_col: object
    range_len: object = field(init=False)

    def __post_init__(self):
        self.range_len = self.max_col - self.min_col + 1


@dataclass
class ValidationReport:
    """Result of `validate_csr` (reference matrix.py:67-75): truthy when the matrix is valid."""

    ok: bool
    message: str = "OK"
    index: int = -1

    def __bool__(self):
        return self.ok


def validate_csr(m: CsrMatrix) -> ValidationReport:
    """First violated CsrMatrix invariant, as a report (reference validate_csr semantics,
    matrix.py:119-150): row_ptr shape / start / monotonicity, col/val lengths, column range,
    and -- for matrices flagged canonical -- strictly increasing columns inside each row."""
    m = m.numpy()
    rp = np.asarray(m.row_ptr, dtype=np.int64)
    if rp.shape != (m.n_rows + 1,):
        return ValidationReport(False, f"row_ptr length {rp.size} != n_rows+1")
    if rp[0] != 0:
        return ValidationReport(False, "row_ptr[0] != 0", 0)
    steps = np.diff(rp)
    bad = np.flatnonzero(steps < 0)
    if bad.size:
        return ValidationReport(False, f"row_ptr decreasing at index {int(bad[0]) + 1}", int(bad[0]) + 1)
    nnz = int(rp[-1])
    col = np.asarray(m.col)
    val = np.asarray(m.val)
    if col.size != nnz or val.size != nnz:
        return ValidationReport(False, f"col/val lengths ({col.size}/{val.size}) != row_ptr[-1] ({nnz})")
    if nnz:
        c = col.astype(np.int64)
        top = int(c.max())
        if top >= m.n_cols:
            at = int(np.flatnonzero(c == top)[0])
            return ValidationReport(False, f"col[{at}] = {top} out of range", at)
        if m.canonical:
            up = np.diff(c) > 0
            starts = rp[1:-1]
            starts = starts[(starts > 0) & (starts < nnz)]
            up[starts - 1] = True          # a new row may start lower
            down = np.flatnonzero(~up)
            if down.size:
                at = int(down[0]) + 1
                return ValidationReport(False, f"columns not strictly increasing within a row at nz {at}", at)
    return ValidationReport(True)


def check_csr(m: CsrMatrix) -> None:
    """validate_csr, raising InputError with the report's message on failure."""
    rep = validate_csr(m)
    if not rep:
        raise InputError(rep.message)


def _col_dtype(n_cols: int):
    """uint32 column indices, uint64 beyond 2^32 columns (reference util.py:47-49)."""
    return np.uint32 if n_cols <= (1 << 32) else np.uint64


def csr_from_arrays(rows, cols, vals, n_rows: int, n_cols: int) -> CsrMatrix:
    """Canonical CSR from coordinate arrays: duplicates summed (in input order), rows sorted
    by column (reference csr_from_arrays matrix.py:77-104)."""
    if n_rows < 0 or n_cols < 0:
        raise InputError("matrix dimensions must be non-negative")
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    v = np.asarray(vals, dtype=np.float64).ravel()
    if r.size == 0:
        return CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, np.int64), np.empty(0, _col_dtype(n_cols)),
                         np.empty(0, np.float64))
    if r.min() < 0 or r.max() >= n_rows:
        raise InputError(f"row index out of range [0, {n_rows})")
    if c.min() < 0 or c.max() >= n_cols:
        raise InputError(f"column index out of range [0, {n_cols})")
    key = r * n_cols + c
    uk, slot = np.unique(key, return_inverse=True)
    sums = np.bincount(slot, weights=v, minlength=uk.size)   # sequential per key, input order
    out_r = uk // n_cols
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(out_r, minlength=n_rows), out=rp[1:])
    return CsrMatrix(n_rows, n_cols, rp, (uk % n_cols).astype(_col_dtype(n_cols)), sums)


def csr_from_triplets(triplets, n_rows: int, n_cols: int) -> CsrMatrix:
    """csr_from_arrays over an iterable of (row, col, val) (reference matrix.py:107-116)."""
    t = list(triplets)
    if not t:
        return csr_from_arrays([], [], [], n_rows, n_cols)
    r, c, v = zip(*t)
    return csr_from_arrays(r, c, v, n_rows, n_cols)


def canonicalize_csr(m: CsrMatrix) -> CsrMatrix:
    """Stable sort of every row by column, in place; the matrix is flagged canonical
    (reference matrix.py:216-224 -- duplicates are kept, not merged)."""
    m2 = m.numpy()
    rp = np.asarray(m2.row_ptr, np.int64)
    if int(rp[-1]):
        rid = np.repeat(np.arange(m2.n_rows, dtype=np.int64), np.diff(rp))
        order = np.lexsort((np.asarray(m2.col), rid))
        m.col = np.asarray(m2.col)[order]
        m.val = np.asarray(m2.val)[order]
        m.row_ptr = rp
    m.canonical = True
    return m


@dataclass
class CscSubMatrix:
    """Column-compressed view of a subset of CSR rows (reference matrix.py:47-63): col_ptr spans
    all columns of the source, `row` holds local row ids into `source_rows`."""

    source_rows: np.ndarray
    n_cols: int
    col_ptr: np.ndarray
    row: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])


def csr_rows_to_csc(source: CsrMatrix, rows) -> CscSubMatrix:
    """Rows `rows` (sorted, unique) of a CSR matrix as a CSC sub-matrix by counting sort:
    inside every column the entries keep ascending local-row order (reference
    csr_rows_to_csc matrix.py:153-184; the order the coarse level's outer product needs)."""
    src = source.numpy()
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size:
        if rows.min() < 0 or rows.max() >= src.n_rows:
            raise InputError("row id out of range")
        if (np.diff(rows) <= 0).any():
            raise InputError("rows must be sorted and unique")
    rp = np.asarray(src.row_ptr, np.int64)
    lo, hi = (rp[rows], rp[rows + 1]) if rows.size else (np.empty(0, np.int64), np.empty(0, np.int64))
    lens = hi - lo
    total = int(lens.sum())
    col_ptr = np.zeros(src.n_cols + 1, np.int64)
    if total == 0:
        return CscSubMatrix(rows, src.n_cols, col_ptr, np.empty(0, np.int64), np.empty(0, np.float64))
    first = np.repeat(lo - np.concatenate(([0], np.cumsum(lens)[:-1])), lens) + np.arange(total)
    c = np.asarray(src.col)[first].astype(np.int64)
    v = np.asarray(src.val)[first]
    local = np.repeat(np.arange(rows.size, dtype=np.int64), lens)
    np.cumsum(np.bincount(c, minlength=src.n_cols), out=col_ptr[1:])
    order = np.argsort(c, kind="stable")       # stable: ascending local row inside each column
    return CscSubMatrix(rows, src.n_cols, col_ptr, local[order], v[order])
