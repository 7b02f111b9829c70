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


def validate_csr(m: CsrMatrix) -> None:
    """Raise InputError on a malformed CSR (reference validate_csr semantics, matrix.py:119-150)."""
    m = m.numpy()
    rp = np.asarray(m.row_ptr, dtype=np.int64)
    if rp.shape != (m.n_rows + 1,):
        raise InputError(f"row_ptr length {rp.size} != n_rows+1")
    if rp[0] != 0:
        raise InputError("row_ptr[0] != 0")
    diffs = np.diff(rp)
    if diffs.size and diffs.min() < 0:
        raise InputError(f"row_ptr decreasing at index {int(np.argmax(diffs < 0)) + 1}")
    nnz = int(rp[-1])
    if len(m.col) != nnz or len(m.val) != nnz:
        raise InputError(f"col/val lengths ({len(m.col)}/{len(m.val)}) != row_ptr[-1] ({nnz})")
    if nnz:
        c = np.asarray(m.col).astype(np.int64)
        if c.min() < 0 or c.max() >= m.n_cols:
            raise InputError("column index out of range")
        if m.canonical:
            inner = np.diff(c)
            idx = rp[1:-1] - 1
            inner[idx[(idx >= 0) & (idx < inner.size)]] = 1
            if inner.size and inner.min() <= 0:
                raise InputError("columns not strictly increasing within a row")
