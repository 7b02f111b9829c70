"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference's own generators (`/root/reference/pkg/src/spgemm/generate.py`)
do not match the BASELINE configs: `gen_rmat` resamples collisions instead of
merging them (generate.py:88-91) and values are 1.0 or (0,1]
(generate.py:98-100,149-150).  These generators follow SURVEY.md §8(d):

* cfg1/cfg4 -- exactly ``d`` distinct uniform columns per row, sorted,
  values U[-1,1];
* cfg2 -- 27-point stencil on a cube, 26.0 on the diagonal, -1.0 off it;
* cfg3/cfg5 -- R-MAT quadrant descent (the same quadrant mapping as
  `_rmat_edge_batch`, generate.py:56-68), duplicates merged, self-loops kept,
  values U[-1,1] drawn after the merge.

Randomness is a counter-based hash (splitmix64 finaliser) of
``(seed, stream, index)``, so the numpy path here and the CUDA path in
``csrc/generate.cu`` produce bit-identical matrices; big configs are built on
the GPU, small ones anywhere.  Everything is host-side setup, not the measured
SpGEMM path.
"""

from __future__ import annotations

import numpy as np

from .matrix import CsrMatrix

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids (shared with csrc/generate.cu)
STREAM_VAL = 0xFF
STREAM_COL = 0xFE


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z + _GOLD
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def hash3(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """64-bit hash of (seed, stream, idx); idx is a uint64 array."""
    with np.errstate(over="ignore"):
        key = _mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) << np.uint64(48)))
        return _mix64(np.asarray(idx, dtype=np.uint64) ^ key)


def uniform01(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) doubles with 53 random bits."""
    h = hash3(seed, stream, idx)
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_pm1(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """U[-1,1) doubles."""
    return 2.0 * uniform01(seed, stream, idx) - 1.0


def uniform_rows(n_rows: int, n_cols: int, d: int, seed: int) -> CsrMatrix:
    """Exactly ``d`` distinct uniform columns per row (Floyd sampling), sorted; U[-1,1] values."""
    if d > n_cols:
        raise ValueError("d must not exceed n_cols")
    rows = np.arange(n_rows, dtype=np.uint64)
    chosen = np.empty((n_rows, d), dtype=np.int64)
    with np.errstate(over="ignore"):
        for s, j in enumerate(range(n_cols - d, n_cols)):
            h = hash3(seed, STREAM_COL, rows * np.uint64(d) + np.uint64(s))
            t = (h % np.uint64(j + 1)).astype(np.int64)
            dup = (chosen[:, :s] == t[:, None]).any(axis=1) if s else np.zeros(n_rows, bool)
            chosen[:, s] = np.where(dup, j, t)
    chosen.sort(axis=1)
    col = chosen.reshape(-1).astype(np.int32)
    row_ptr = (np.arange(n_rows + 1, dtype=np.int64) * d).astype(np.int64)
    val = uniform_pm1(seed, STREAM_VAL, np.arange(col.size, dtype=np.uint64))
    return CsrMatrix(n_rows, n_cols, row_ptr, col, val)


def stencil27(g: int) -> CsrMatrix:
    """27-point stencil on a g^3 grid (row = (x*g + y)*g + z); 26 on the diagonal, -1 off it."""
    n = g * g * g
    r = np.arange(n, dtype=np.int64)
    x, y, z = r // (g * g), (r // g) % g, r % g
    cols, vals, lens = [], [], np.zeros(n, dtype=np.int64)
    offs = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)]
    # offsets enumerate in ascending column order because col = r + dx*g*g + dy*g + dz
    mask_all = []
    for dx, dy, dz in offs:
        ok = (x + dx >= 0) & (x + dx < g) & (y + dy >= 0) & (y + dy < g) & (z + dz >= 0) & (z + dz < g)
        mask_all.append(ok)
        lens += ok
    M = np.stack(mask_all, axis=1)  # n x 27, column order ascending
    C = r[:, None] + np.array([dx * g * g + dy * g + dz for dx, dy, dz in offs])[None, :]
    V = np.where(np.array([o == (0, 0, 0) for o in offs])[None, :], 26.0, -1.0) * np.ones((n, 1))
    col = C[M].astype(np.int32)
    val = V[M].astype(np.float64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    return CsrMatrix(n, n, row_ptr, col, val)


def rmat_edges(scale: int, n_edges: int, seed: int, a=0.57, b=0.19, c=0.19, lo: int = 0):
    """Edges ``lo .. lo+n_edges`` of the R-MAT stream: one U[0,1) draw per level."""
    e = np.arange(lo, lo + n_edges, dtype=np.uint64)
    rows = np.zeros(n_edges, dtype=np.int64)
    cols = np.zeros(n_edges, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for lvl in range(scale):
        u = uniform01(seed, lvl, e)
        row_bit = u >= ab
        col_bit = ((u >= a) & (u < ab)) | (u >= abc)
        rows = (rows << 1) | row_bit
        cols = (cols << 1) | col_bit
    return rows, cols


def rmat(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19) -> CsrMatrix:
    """R-MAT with duplicates merged (self-loops kept), U[-1,1] values drawn after the merge."""
    n = 1 << scale
    m = edge_factor * n
    keys = []
    step = 1 << 24
    for lo in range(0, m, step):
        r, c_ = rmat_edges(scale, min(step, m - lo), seed, a, b, c, lo)
        keys.append(np.unique(r * n + c_))
    key = np.unique(np.concatenate(keys))
    rows = key // n
    col = (key % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    val = uniform_pm1(seed, STREAM_VAL, np.arange(col.size, dtype=np.uint64))
    return CsrMatrix(n, n, row_ptr, col, val)


# BASELINE.json configs (seeds recorded in DESIGN.md)
CONFIGS = {
    1: dict(kind="uniform", n=16384, d=16, seed=1, product="AA"),
    2: dict(kind="stencil", g=64, product="AA"),
    3: dict(kind="rmat", scale=20, ef=16, seed=3, product="AA"),
    4: dict(kind="uniform", n=1 << 23, d=8, seed=4, seed_b=40, product="AB"),
    5: dict(kind="rmat", scale=24, ef=32, seed=5, product="AA"),
}


def make_config_cpu(cfg: int):
    """(A, B) for a config, generated with numpy (cfg5 is too big for this path)."""
    p = CONFIGS[cfg]
    if p["kind"] == "uniform":
        A = uniform_rows(p["n"], p["n"], p["d"], p["seed"])
        B = uniform_rows(p["n"], p["n"], p["d"], p["seed_b"]) if p["product"] == "AB" else A
    elif p["kind"] == "stencil":
        A = stencil27(p["g"])
        B = A
    else:
        A = rmat(p["scale"], p["ef"], p["seed"])
        B = A
    return A, B


# ------------------------------------------------------------------ device path
def _gen_lib():
    from . import _lib
    return _lib.lib()


def _seed_key(seed: int) -> int:
    return int(seed) & 0xFFFFFFFFFFFFFFFF


def rmat_device(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19, device="cuda", rp_dtype=None):
    """Same matrix as `rmat` (bit-identical), built on the GPU; returns a CsrMatrix of CUDA tensors."""
    import ctypes as C

    import torch

    L = _gen_lib()
    n = 1 << scale
    m = edge_factor * n
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    keys = torch.empty(m, dtype=torch.int64, device=device)
    step = 1 << 28
    for lo in range(0, m, step):
        cnt = min(step, m - lo)
        rc = L.magnus_gen_rmat_keys(scale, lo, cnt, _seed_key(seed), a, b, c, C.c_void_p(keys.data_ptr() + lo * 8), stream)
        assert rc == 0
    keys = torch.unique(keys, sorted=True)          # merge duplicates (self-loops kept)
    rows = keys >> scale
    col = (keys & (n - 1)).to(torch.int32)
    del keys
    counts = torch.bincount(rows, minlength=n)
    del rows
    rp = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=rp[1:])
    if rp_dtype is not None:
        rp = rp.to(rp_dtype)
    val = torch.empty(col.numel(), dtype=torch.float64, device=device)
    assert L.magnus_gen_uniform_pm1(_seed_key(seed), STREAM_VAL, col.numel(), C.c_void_p(val.data_ptr()), stream) == 0
    return CsrMatrix(n, n, rp, col, val)


def uniform_rows_device(n_rows: int, n_cols: int, d: int, seed: int, device="cuda", rp_dtype=None):
    """Same matrix as `uniform_rows`, built on the GPU."""
    import ctypes as C

    import torch

    L = _gen_lib()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    col = torch.empty(n_rows * d, dtype=torch.int32, device=device)
    assert L.magnus_gen_uniform_rows(n_rows, n_cols, d, _seed_key(seed), C.c_void_p(col.data_ptr()), stream) == 0
    rp = torch.arange(n_rows + 1, dtype=torch.int64, device=device) * d
    if rp_dtype is not None:
        rp = rp.to(rp_dtype)
    val = torch.empty(n_rows * d, dtype=torch.float64, device=device)
    assert L.magnus_gen_uniform_pm1(_seed_key(seed), STREAM_VAL, n_rows * d, C.c_void_p(val.data_ptr()), stream) == 0
    return CsrMatrix(n_rows, n_cols, rp, col, val)


def stencil27_device(g: int, device="cuda", rp_dtype=None):
    import torch
    m = stencil27(g)
    rp = torch.from_numpy(m.row_ptr).to(device)
    if rp_dtype is not None:
        rp = rp.to(rp_dtype)
    return CsrMatrix(m.n_rows, m.n_cols, rp, torch.from_numpy(m.col).to(device), torch.from_numpy(m.val).to(device))


def make_config_device(cfg: int, rp_dtype=None):
    """(A, B) of a BASELINE config as CUDA tensors (cfg3: row_ptr int32 per BASELINE unless given)."""
    p = CONFIGS[cfg]
    if p["kind"] == "uniform":
        A = uniform_rows_device(p["n"], p["n"], p["d"], p["seed"], rp_dtype=rp_dtype)
        B = uniform_rows_device(p["n"], p["n"], p["d"], p["seed_b"], rp_dtype=rp_dtype) if p["product"] == "AB" else A
    elif p["kind"] == "stencil":
        A = stencil27_device(p["g"], rp_dtype=rp_dtype)
        B = A
    else:
        A = rmat_device(p["scale"], p["ef"], p["seed"], rp_dtype=rp_dtype)
        B = A
    return A, B
