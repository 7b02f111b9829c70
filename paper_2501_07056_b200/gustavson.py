"""Gustavson baselines on the device -- reference gustavson.py:155-268.

The reference ships two non-MAGNUS pipelines next to `spgemm_magnus`: a
Gustavson SpGEMM with a full-width dense accumulator and an
expand-sort-compress (ESC) one, both behind the same symbolic pass.  They are
the ablation that shows what MAGNUS's locality generation buys, and a second
path the MAGNUS result can be checked against.  Same names, arguments, result
type and counters as the reference:

    gustavson_dense_symbolic(A, B, threads=1) -> row_ptr (int64, n_rows+1)
    gustavson_dense_numeric(A, B, row_ptr, threads=1) -> SpgemmResult
    gustavson_esc_numeric(A, B, row_ptr, threads=1) -> SpgemmResult
    gustavson_dense(A, B, threads=1) / gustavson_esc(A, B, threads=1) -> SpgemmResult

Values follow the reference bit for bit: dense = sequential from +0.0 in
Gustavson order (DenseAccumulator), ESC = x0 + pairwise(rest)
(sort_accumulate).  Kernels: csrc/baselines.cuh behind the C-ABI
`magnus_gd_*` / `magnus_esc_*`; the ESC sort step is the library's own stable
LSD radix sort (csrc/radix_sort.cuh; MAGNUS_ESC_SORT=cub selects torch.sort).
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os as _os
import time

import numpy as np

from . import _lib
from .errors import ContractViolation, OverBudgetError
from .magnus import SpgemmResult, _abi, _check_dims, _is_host, _to_device, _torch
from .matrix import CsrMatrix

ESC_BATCH_PRODUCTS = 1 << 27   # products expanded and sorted per ESC batch (~5 GB of keys, values, sort buffers)


class _Pair:
    """A, B on the device plus their C-ABI views."""

    def __init__(self, A, B):
        torch = _torch()
        _check_dims(A, B)
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.host_io = _is_host(A)
        self.A = _to_device(A, self.device)
        self.B = self.A if B is A else _to_device(B, self.device)
        self.a, self.b = _abi(self.A), _abi(self.B)
        self.stream = torch.cuda.current_stream(self.device)

    def sp(self):
        return C.c_void_p(self.stream.cuda_stream)

    def scratch(self):
        """Dense-accumulator scratch: up to 4 rows per SM, at most a quarter of free memory."""
        torch = self.torch
        per = int(_lib.lib().magnus_gd_scratch_bytes(max(self.B.n_cols, 1), 1))
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        free, _ = torch.cuda.mem_get_info(self.device)
        nbytes = min(per * sms * 4, max(per, free // 4))
        nbytes = min(nbytes, per * max(self.A.n_rows, 1))
        return torch.empty(nbytes + 16, dtype=torch.uint8, device=self.device)

    def inter_offsets(self):
        """Exclusive prefix of the rows' product counts (row_intermediate_stats gustavson.py:97-134)."""
        torch = self.torch
        n = self.A.n_rows
        inter = torch.empty(n, dtype=torch.int64, device=self.device)
        mn = torch.empty(n, dtype=torch.int64, device=self.device)
        mx = torch.empty(n, dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().magnus_row_stats(C.byref(self.a), C.byref(self.b), C.c_void_p(inter.data_ptr()),
                                               C.c_void_p(mn.data_ptr()), C.c_void_p(mx.data_ptr()), self.sp()))
        off = torch.zeros(n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(inter, 0, out=off[1:])
        return off

    def result(self, rp, col, val, timings, counters):
        if self.host_io:
            return SpgemmResult(CsrMatrix(self.A.n_rows, self.B.n_cols, rp.cpu().numpy(), col.cpu().numpy().view(np.uint32),
                                          val.cpu().numpy(), canonical=True), timings, counters)
        return SpgemmResult(CsrMatrix(self.A.n_rows, self.B.n_cols, rp, col, val, canonical=True), timings, counters)


def _device_row_ptr(P: _Pair, row_ptr):
    torch = P.torch
    rp = torch.as_tensor(np.asarray(row_ptr) if isinstance(row_ptr, np.ndarray) else row_ptr)
    if tuple(rp.shape) != (P.A.n_rows + 1,) or int(rp[0]) != 0:
        raise ContractViolation("row_ptr does not come from a symbolic pass of (A, B)")
    return rp.to(P.device, torch.int64).contiguous()


def _symbolic(P: _Pair):
    torch = P.torch
    rp = torch.empty(P.A.n_rows + 1, dtype=torch.int64, device=P.device)
    scratch = P.scratch()
    _lib.check(_lib.lib().magnus_gd_symbolic(C.byref(P.a), C.byref(P.b), C.c_void_p(rp.data_ptr()),
                                             C.c_void_p(scratch.data_ptr()), scratch.numel(), P.sp()))
    return rp


def gustavson_dense_symbolic(A: CsrMatrix, B: CsrMatrix, threads: int = 1):
    """Precise-prediction symbolic phase: exact per-row nnz, prefix-summed (gustavson.py:155-170)."""
    P = _Pair(A, B)
    rp = _symbolic(P)
    return rp.cpu().numpy() if P.host_io else rp


def _inter_total(P: _Pair) -> int:
    return int(P.inter_offsets()[-1])


def _dense_numeric(P: _Pair, rp):
    torch = P.torch
    nnz = int(rp[-1])
    col = torch.empty(nnz, dtype=torch.int32, device=P.device)
    val = torch.empty(nnz, dtype=torch.float64, device=P.device)
    scratch = P.scratch()
    _lib.check(_lib.lib().magnus_gd_numeric(C.byref(P.a), C.byref(P.b), C.c_void_p(rp.data_ptr()),
                                            C.c_void_p(col.data_ptr()), C.c_void_p(val.data_ptr()),
                                            C.c_void_p(scratch.data_ptr()), scratch.numel(), P.sp()))
    return col, val


def gustavson_dense_numeric(A: CsrMatrix, B: CsrMatrix, row_ptr, threads: int = 1) -> SpgemmResult:
    """Numeric phase with a full-width dense accumulator (gustavson.py:184-220).  The device emits
    rows sorted, so the reference's separate canonicalisation ('post') costs nothing here."""
    P = _Pair(A, B)
    rp = _device_row_ptr(P, row_ptr)
    t0 = time.perf_counter()
    col, val = _dense_numeric(P, rp)
    P.stream.synchronize()
    t1 = time.perf_counter()
    counters = {"inter_prod_size": _inter_total(P), "nnz_c": int(rp[-1])}
    return P.result(rp, col, val, {"numeric": t1 - t0, "post": 0.0}, counters)


def _esc_numeric(P: _Pair, rp, batch_products: int = ESC_BATCH_PRODUCTS):
    torch = P.torch
    nnz = int(rp[-1])
    n = P.A.n_rows
    col = torch.empty(nnz, dtype=torch.int32, device=P.device)
    val = torch.empty(nnz, dtype=torch.float64, device=P.device)
    off = P.inter_offsets()
    total = int(off[-1])
    off_h = off.cpu().numpy()
    rp_h = rp.cpu().numpy()
    L = _lib.lib()
    r0 = 0
    while r0 < n:
        # largest contiguous row range whose products fit the batch (at least one row)
        r1 = int(np.searchsorted(off_h, off_h[r0] + batch_products, side="right")) - 1
        r1 = min(max(r1, r0 + 1), n, r0 + (1 << 31))
        m = int(off_h[r1] - off_h[r0])
        if m > 4 * batch_products:
            free, _ = torch.cuda.mem_get_info(P.device)
            if m * 48 > free:
                raise OverBudgetError(f"row {r0}: buffering {m} products exceeds the device memory budget")
        if m:
            keys = torch.empty(m, dtype=torch.int64, device=P.device)
            vals = torch.empty(m, dtype=torch.float64, device=P.device)
            _lib.check(L.magnus_esc_expand(C.byref(P.a), C.byref(P.b), r0, r1, C.c_void_p(off.data_ptr()),
                                           C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()), P.sp()))
            # stable sort by (row, column): the library's own LSD radix sort over the key bytes that can differ
            # (MAGNUS_ESC_SORT=cub: torch.sort)
            if _os.environ.get("MAGNUS_ESC_SORT") == "cub":
                skeys, perm = torch.sort(keys, stable=True)
            else:
                mask = ((1 << max(1, int(P.B.n_cols - 1).bit_length())) - 1) | (((1 << max(1, int(r1 - r0 - 1).bit_length())) - 1) << 32)
                skeys, perm = _lib.sort_pairs(keys, key_mask=mask)
            del keys
            run = torch.empty(m + 1, dtype=torch.int64, device=P.device)
            runs = C.c_int64(0)
            want = int(rp_h[r1] - rp_h[r0])
            # count the runs first: a mismatch must not write outside the batch's rows
            _lib.check(L.magnus_esc_compress(C.c_void_p(skeys.data_ptr()), C.c_void_p(perm.data_ptr()),
                                             C.c_void_p(vals.data_ptr()), m, 0, None, None, C.c_void_p(run.data_ptr()),
                                             C.byref(runs), P.sp()))
            if runs.value != want:
                raise ContractViolation(f"rows {r0}..{r1 - 1}: symbolic predicted {want} nnz, numeric produced {runs.value}")
            _lib.check(L.magnus_esc_compress(C.c_void_p(skeys.data_ptr()), C.c_void_p(perm.data_ptr()),
                                             C.c_void_p(vals.data_ptr()), m, int(rp_h[r0]), C.c_void_p(col.data_ptr()),
                                             C.c_void_p(val.data_ptr()), C.c_void_p(run.data_ptr()), C.byref(runs),
                                             P.sp()))
            del skeys, perm, vals, run
        elif rp_h[r1] != rp_h[r0]:
            raise ContractViolation(f"rows {r0}..{r1 - 1}: symbolic predicted nonzeros for an empty product")
        r0 = r1
    return col, val, total


def gustavson_esc_numeric(A: CsrMatrix, B: CsrMatrix, row_ptr, threads: int = 1) -> SpgemmResult:
    """Numeric phase via expand-sort-compress (gustavson.py:223-250)."""
    P = _Pair(A, B)
    rp = _device_row_ptr(P, row_ptr)
    t0 = time.perf_counter()
    col, val, total = _esc_numeric(P, rp)
    P.stream.synchronize()
    t1 = time.perf_counter()
    return P.result(rp, col, val, {"numeric": t1 - t0, "post": 0.0}, {"inter_prod_size": total, "nnz_c": int(rp[-1])})


def _pipeline(A, B, esc: bool) -> SpgemmResult:
    """_timed_pipeline gustavson.py:253-259: dense symbolic, then the numeric phase."""
    P = _Pair(A, B)
    t0 = time.perf_counter()
    rp = _symbolic(P)
    P.stream.synchronize()
    t1 = time.perf_counter()
    if esc:
        col, val, total = _esc_numeric(P, rp)
    else:
        col, val = _dense_numeric(P, rp)
        total = None
    P.stream.synchronize()
    t2 = time.perf_counter()
    if total is None:
        total = _inter_total(P)
    timings = {"setup": 0.0, "symbolic": t1 - t0, "numeric": t2 - t1, "post": 0.0}
    return P.result(rp, col, val, timings, {"inter_prod_size": total, "nnz_c": int(rp[-1])})


def gustavson_dense(A: CsrMatrix, B: CsrMatrix, threads: int = 1) -> SpgemmResult:
    """Symbolic + numeric dense-accumulation Gustavson pipeline (gustavson.py:262-264)."""
    return _pipeline(A, B, esc=False)


def gustavson_esc(A: CsrMatrix, B: CsrMatrix, threads: int = 1) -> SpgemmResult:
    """Symbolic + numeric expand-sort-compress pipeline (gustavson.py:267-268)."""
    return _pipeline(A, B, esc=True)
