"""Matrix files: Matrix Market coordinate text and the SPGC binary cache.

Same functions, file formats and errors as the reference's mmio.py (1-189):

* ``read_matrix_market(path)`` -- coordinate format, fields real / integer /
  pattern / complex (integer and complex coerced to real, complex keeps the real
  part, pattern entries are 1.0), symmetries general / symmetric /
  skew-symmetric / hermitian (expanded to full storage: mirrored off-diagonal
  entries appended, negated for skew-symmetric); array format rejected;
  duplicates summed; rows sorted -- a canonical CsrMatrix.  Malformed input
  raises ``ParseError`` with the 1-based line number.
* ``write_matrix_market(m, path, comment=None)`` -- ``coordinate real general``,
  1-based, values printed with 17 significant digits.
* ``write_binary_cache`` / ``read_binary_cache`` -- the SPGC layout
  (little endian): 40-byte header ``b"SPGC"``, version u32 = 1, n_rows,
  n_cols, nnz (u64), column width (4 or 8), value width (8), canonical flag,
  5 zero bytes; then row_ptr int64[n_rows+1], col u32/u64[nnz], val f64[nnz].
* ``read_matrix`` / ``write_matrix`` -- ``.bin`` / ``.spgc`` is the cache,
  anything else Matrix Market.

B200 additions: ``read_binary_cache(path, device="cuda")`` reads the three
arrays straight into page-locked host buffers and copies them to the device
(int64 row_ptr, int32 col, f64 val -- what ``spgemm_magnus`` consumes), so a
cached input reaches HBM at PCIe speed without a numpy detour; the writers
accept device matrices.  Host-side plumbing -- not on the SpGEMM path.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import InputError, ParseError
from .matrix import CsrMatrix

SPGC_MAGIC = b"SPGC"
SPGC_VERSION = 1
_HEADER = struct.Struct("<4sIQQQBBB5x")   # 40 bytes

_FIELDS = ("real", "integer", "pattern", "complex")
_SYMMETRIES = ("general", "symmetric", "skew-symmetric", "hermitian")


def col_dtype(n_cols: int):
    """uint32 column indices up to 2^32 columns, uint64 beyond (reference util.py:47-49)."""
    return np.uint32 if n_cols <= 1 << 32 else np.uint64


def _host(x):
    if isinstance(x, np.ndarray):
        return x
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def csr_from_coo(rows, cols, vals, n_rows: int, n_cols: int) -> CsrMatrix:
    """Canonical CSR from coordinates: rows sorted by column, duplicates summed sequentially in input
    order (the reference's csr_from_arrays, matrix.py:76-104: np.unique + np.bincount)."""
    if n_rows < 0 or n_cols < 0:
        raise InputError("matrix dimensions must be non-negative")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    cd = col_dtype(n_cols)
    if rows.size == 0:
        return CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, np.int64), np.empty(0, cd), np.empty(0, np.float64), True)
    if rows.min() < 0 or rows.max() >= n_rows:
        raise InputError(f"row index out of range [0, {n_rows})")
    if cols.min() < 0 or cols.max() >= n_cols:
        raise InputError(f"column index out of range [0, {n_cols})")
    order = np.lexsort((cols, rows))
    r_s, c_s = rows[order], cols[order]
    head = np.ones(order.size, bool)
    head[1:] = (r_s[1:] != r_s[:-1]) | (c_s[1:] != c_s[:-1])
    run_sorted = np.cumsum(head) - 1
    run = np.empty_like(run_sorted)
    run[order] = run_sorted                      # run id of every input entry, in input order
    nrun = int(run_sorted[-1]) + 1
    summed = np.bincount(run, weights=vals, minlength=nrun)   # sequential from 0.0, input order
    out_r, out_c = r_s[head], c_s[head]
    row_ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(out_r, minlength=n_rows), out=row_ptr[1:])
    return CsrMatrix(n_rows, n_cols, row_ptr, out_c.astype(cd), summed, True)


# ---------------------------------------------------------------- Matrix Market
def read_matrix_market(path) -> CsrMatrix:
    with open(path, "r", encoding="latin-1") as f:
        text = f.read().splitlines()
    if not text:
        raise ParseError("empty file", line=1)
    banner = text[0].split()
    if len(banner) != 5 or banner[0].lower() != "%%matrixmarket":
        raise ParseError("expected '%%MatrixMarket matrix coordinate <field> <symmetry>'", line=1)
    obj, fmt, field, sym = (t.lower() for t in banner[1:])
    if obj != "matrix":
        raise ParseError(f"unsupported object '{obj}'", line=1)
    if fmt == "array":
        raise ParseError("array (dense) format is not supported", line=1)
    if fmt != "coordinate":
        raise ParseError(f"unsupported format '{fmt}'", line=1)
    if field not in _FIELDS:
        raise ParseError(f"unsupported field '{field}'", line=1)
    if sym not in _SYMMETRIES:
        raise ParseError(f"unsupported symmetry '{sym}'", line=1)

    # data lines (1-based line numbers kept for errors); the first one is the size line
    lines = [(no, s) for no, s in ((i + 1, raw.strip()) for i, raw in enumerate(text)) if no > 1 and s and s[0] != "%"]
    if not lines:
        raise ParseError("missing dimension line", line=len(text))
    size_no, size_line = lines[0]
    parts = size_line.split()
    if len(parts) != 3:
        raise ParseError(f"expected 'rows cols nnz', got {size_line!r}", line=size_no)
    try:
        n_rows, n_cols, nnz = (int(p) for p in parts)
    except ValueError:
        raise ParseError(f"non-integer dimension in {size_line!r}", line=size_no) from None
    if min(n_rows, n_cols, nnz) < 0:
        raise ParseError("negative dimension", line=size_no)

    body = lines[1:]
    if len(body) > nnz:
        raise ParseError(f"more than the declared {nnz} entries", line=body[nnz][0])
    want = {"pattern": 2, "complex": 4}.get(field, 3)
    toks = [s.split() for _, s in body]
    for (no, s), t in zip(body, toks):
        if len(t) != want:
            raise ParseError(f"expected {want} fields, got {len(t)}", line=no)
    if len(body) != nnz:
        raise ParseError(f"declared {nnz} entries but found {len(body)}", line=len(text))
    try:
        arr = np.array([t[:2] for t in toks], dtype=np.int64).reshape(-1, 2)
        vals = np.ones(nnz) if field == "pattern" else np.array([t[2] for t in toks], dtype=np.float64)
    except (ValueError, OverflowError):
        for (no, s), t in zip(body, toks):   # locate the offending line
            try:
                int(t[0]), int(t[1])
                if field != "pattern":
                    float(t[2])
            except (ValueError, OverflowError):
                raise ParseError(f"malformed entry {s!r}", line=no) from None
        raise
    r, c = arr[:, 0], arr[:, 1]
    bad = np.nonzero((r < 1) | (r > n_rows) | (c < 1) | (c > n_cols))[0]
    if bad.size:
        no = body[int(bad[0])][0]
        raise ParseError(f"index ({int(r[bad[0]])}, {int(c[bad[0]])}) outside {n_rows} x {n_cols}", line=no)
    r, c = r - 1, c - 1
    if sym != "general":
        off = r != c
        mirror_v = -vals[off] if sym == "skew-symmetric" else vals[off]
        r, c, vals = np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([vals, mirror_v])
    return csr_from_coo(r, c, vals, n_rows, n_cols)


def write_matrix_market(m: CsrMatrix, path, comment: str = None) -> None:
    rp = _host(m.row_ptr).astype(np.int64)
    col = _host(m.col)
    col = (col.view(np.uint32) if col.dtype == np.int32 else col).astype(np.int64)
    val = _host(m.val).astype(np.float64)
    rows = np.repeat(np.arange(m.n_rows, dtype=np.int64), np.diff(rp))
    with open(path, "w", encoding="ascii") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        for line in (comment.splitlines() if comment else []):
            f.write(f"% {line}\n")
        f.write(f"{m.n_rows} {m.n_cols} {rows.size}\n")
        f.writelines(f"{i} {j} {v:.17g}\n" for i, j, v in zip((rows + 1).tolist(), (col + 1).tolist(), val.tolist()))


# ---------------------------------------------------------------- SPGC binary cache
def write_binary_cache(m: CsrMatrix, path) -> None:
    rp = _host(m.row_ptr).astype("<i8", copy=False)
    col = _host(m.col)
    if col.dtype in (np.int32, np.uint32):
        col = col.view(np.uint32)
    width = 8 if (col.dtype.itemsize == 8 and m.n_cols > 1 << 32) else 4
    col = col.astype(f"<u{width}", copy=False)
    val = _host(m.val).astype("<f8", copy=False)
    hdr = _HEADER.pack(SPGC_MAGIC, SPGC_VERSION, m.n_rows, m.n_cols, int(col.size), width, 8, int(bool(m.canonical)))
    with open(path, "wb") as f:
        f.write(hdr)
        for a in (rp, col, val):
            f.write(np.ascontiguousarray(a).data)


def _read_header(f, size):
    raw = f.read(_HEADER.size)
    if len(raw) < _HEADER.size or raw[:4] != SPGC_MAGIC:
        raise ParseError("not a binary cache file (bad magic)")
    _, version, n_rows, n_cols, nnz, cw, vw, canon = _HEADER.unpack(raw)
    if version != SPGC_VERSION:
        raise ParseError(f"unsupported cache version {version}")
    if cw not in (4, 8) or vw != 8:
        raise ParseError(f"unsupported widths col={cw} val={vw}")
    need = _HEADER.size + (n_rows + 1) * 8 + nnz * (cw + 8)
    if size != need:
        raise ParseError(f"truncated cache file: {size} bytes, expected {need}")
    return int(n_rows), int(n_cols), int(nnz), cw, bool(canon)


def read_binary_cache(path, device=None) -> CsrMatrix:
    """SPGC file -> CsrMatrix (numpy; col uint32/uint64 by n_cols).  device="cuda[:i]": int64 row_ptr,
    int32 col and f64 val device tensors, read through page-locked host buffers."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        n_rows, n_cols, nnz, cw, canon = _read_header(f, size)
        if device is None:
            rp = np.fromfile(f, dtype="<i8", count=n_rows + 1).astype(np.int64, copy=False)
            col = np.fromfile(f, dtype=f"<u{cw}", count=nnz).astype(col_dtype(n_cols), copy=False)
            val = np.fromfile(f, dtype="<f8", count=nnz).astype(np.float64, copy=False)
            return CsrMatrix(n_rows, n_cols, rp, col, val, canon)
        import torch

        if cw != 4:
            raise InputError("device matrices hold 32-bit column indices (n_cols <= 2^32)")
        out = []
        for count, dt in ((n_rows + 1, torch.int64), (nnz, torch.int32), (nnz, torch.float64)):
            h = torch.empty(count, dtype=dt, pin_memory=True)
            if count:
                f.readinto(memoryview(h.numpy()).cast("B"))
            out.append(h.to(device, non_blocking=True))
        torch.cuda.current_stream(torch.device(device)).synchronize()
        return CsrMatrix(n_rows, n_cols, out[0], out[1], out[2], canon)


def _is_cache(path) -> bool:
    return str(path).endswith((".bin", ".spgc"))


def read_matrix(path, device=None) -> CsrMatrix:
    """`.bin` / `.spgc`: binary cache; anything else: Matrix Market."""
    if _is_cache(path):
        return read_binary_cache(path, device=device)
    m = read_matrix_market(path)
    if device is not None:
        from .magnus import _to_device
        import torch

        m = _to_device(m, torch.device(device))
    return m


def write_matrix(m: CsrMatrix, path) -> None:
    (write_binary_cache if _is_cache(path) else write_matrix_market)(m, path)
