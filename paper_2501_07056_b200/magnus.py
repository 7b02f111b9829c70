"""`spgemm_magnus` -- drop-in for the reference's entry point (magnus.py:545-583).

Same name, keyword API, result type and error classes as the reference:

    spgemm_magnus(A, B, sys=None, thresholds=None, threads=1, force_fine_only=False) -> SpgemmResult

`A`/`B` are `CsrMatrix` objects whose arrays are numpy (host; the reference's
own representation -- C comes back as numpy, col uint32 like the reference)
or torch tensors (CUDA tensors stay on the device; C comes back on the device).
The computation is the sm_100a CUDA path behind include/magnus_b200.h; there
is no CPU fallback.

`sys=None` probes the device (`detect_device_params`: 227 KB shared memory per
block plays the role of the reference's per-core L2).  Passing the reference's
host `SystemParams` instead reproduces the reference's result for that
configuration bit for bit: categories, and with them the summation
association of every value, follow `sys` exactly as in the reference.
`threads` is accepted for API compatibility; the device decides its own
parallelism.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .accumulators import AccumThresholds
from .errors import ContractViolation, InputError
from .matrix import CsrMatrix, RowStats
from .planner import NUMERIC, SYMBOLIC, SystemParams, compute_chunk_plan, detect_device_params


@dataclass
class SpgemmResult:
    """Reference gustavson.py:28-36."""

    C: CsrMatrix
    phase_timings: dict = field(default_factory=dict)
    counters: dict = field(default_factory=dict)

    @property
    def total_seconds(self) -> float:
        return sum(self.phase_timings.values())


@dataclass
class RowCategories:
    """Reference magnus.py:51-65 (row lists, ascending)."""

    sort_rows: object
    dense_rows: object
    fine_rows: object
    coarse_rows: object

    @property
    def counts(self) -> dict:
        return {"sort": int(len(self.sort_rows)), "dense": int(len(self.dense_rows)),
                "fine": int(len(self.fine_rows)), "coarse": int(len(self.coarse_rows))}


def _torch():
    import torch
    return torch


def _is_host(m: CsrMatrix) -> bool:
    if isinstance(m.row_ptr, np.ndarray):
        return True
    return not m.row_ptr.is_cuda


def _to_device(m: CsrMatrix, device):
    """Device CsrMatrix (torch tensors) + the magnus_csr view of it."""
    torch = _torch()

    def dev(x, dtype):
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.dtype != dtype:
            x = x.to(dtype)
        return x.to(device, non_blocking=True).contiguous()

    rp = m.row_ptr
    rp_dtype = torch.int32 if (getattr(rp, "dtype", None) in (np.int32, torch.int32)) else torch.int64
    rp_t = dev(rp, rp_dtype)
    col = m.col
    if isinstance(col, np.ndarray):
        col = col.view(np.int32) if col.dtype in (np.uint32, np.int32) else col.astype(np.int32)
    col_t = dev(col, torch.int32)
    val_t = dev(m.val, torch.float64)
    d = CsrMatrix(m.n_rows, m.n_cols, rp_t, col_t, val_t, m.canonical)
    return d


def _abi(d: CsrMatrix) -> _lib.Csr:
    nnz = int(d.col.numel())
    return _lib.Csr(d.n_rows, d.n_cols, nnz, d.row_ptr.data_ptr(), d.row_ptr.element_size(), d.col.data_ptr(),
                    d.val.data_ptr())


def _sys_abi(sys: SystemParams) -> _lib.Sys:
    return _lib.Sys(sys.cache_line_bytes, sys.l2_bytes, sys.memory_budget_bytes, sys.histo_type_bytes,
                    sys.prefix_sum_type_bytes, sys.val_bytes)


def _check_dims(A, B):
    """Reference gustavson.py:39-41."""
    if A.n_cols != B.n_rows:
        raise InputError(f"dimension mismatch: A is {A.n_rows}x{A.n_cols}, B is {B.n_rows}x{B.n_cols}")


class MagnusPlan:
    """Device state between the phases (what the reference passes around as
    ``plan_sym, plan_num, cats, stats`` -- magnus.py:568-575)."""

    def __init__(self, A, B, sys=None, thresholds=None, force_fine_only=False, stream=None):
        torch = _torch()
        _check_dims(A, B)
        self.sys = sys if sys is not None else detect_device_params()
        self.thresholds = thresholds if thresholds is not None else AccumThresholds()
        self.force_fine_only = bool(force_fine_only)
        m_c = max(B.n_cols, 1)
        self.plan_sym = compute_chunk_plan(self.sys, m_c, SYMBOLIC, allow_coarse=not force_fine_only)
        self.plan_num = compute_chunk_plan(self.sys, m_c, NUMERIC, allow_coarse=not force_fine_only)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.host_io = _is_host(A)
        self.A = _to_device(A, self.device)
        self.B = self.A if B is A else _to_device(B, self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ctx = _lib.Context()
        self._a, self._b = _abi(self.A), _abi(self.B)
        th = _lib.Thresholds(self.thresholds.sort_dense_crossover, self.thresholds.sort_sweet_spot)
        _lib.check(_lib.lib().magnus_setup(self.ctx.h, C.byref(self._a), C.byref(self._b), C.byref(_sys_abi(self.sys)),
                                           C.byref(th), int(self.force_fine_only), C.c_void_p(self.stream.cuda_stream)))
        self.row_ptr = None
        self.nnz = None

    def reset(self, A) -> None:
        """Re-plan for another A (same B, parameters and stream) on the same context: the
        B-derived device state (validation, skip list, window index) is kept.  Used by the
        row waves of products whose C cannot be held at once (waves.py)."""
        _check_dims(A, self.B)
        self.A = _to_device(A, self.device)
        self._a = _abi(self.A)
        th = _lib.Thresholds(self.thresholds.sort_dense_crossover, self.thresholds.sort_sweet_spot)
        _lib.check(_lib.lib().magnus_setup(self.ctx.h, C.byref(self._a), C.byref(self._b), C.byref(_sys_abi(self.sys)),
                                           C.byref(th), int(self.force_fine_only), C.c_void_p(self.stream.cuda_stream)))
        self.row_ptr = None
        self.nnz = None

    def categories(self) -> RowCategories:
        torch = _torch()
        cat = torch.empty(self.A.n_rows, dtype=torch.int8, device=self.device)
        _lib.check(_lib.lib().magnus_categories(self.ctx.h, C.c_void_p(cat.data_ptr()), C.c_void_p(self.stream.cuda_stream)))
        lists = [torch.nonzero(cat == c).flatten() for c in range(4)]
        return RowCategories(*lists)

    def symbolic(self):
        """magnus_symbolic (reference magnus.py:420-456): exact C.row_ptr (int64)."""
        torch = _torch()
        rp = torch.empty(self.A.n_rows + 1, dtype=torch.int64, device=self.device)
        nnz = C.c_int64(0)
        _lib.check(_lib.lib().magnus_symbolic(self.ctx.h, C.c_void_p(rp.data_ptr()), C.byref(nnz),
                                              C.c_void_p(self.stream.cuda_stream)))
        self.row_ptr, self.nnz = rp, int(nnz.value)
        return rp

    def workspace_bytes(self):
        """(preferred, minimum) device bytes of the numeric phase's reorder buffer (after symbolic)."""
        pref, mini = C.c_int64(0), C.c_int64(0)
        _lib.check(_lib.lib().magnus_workspace_bytes(self.ctx.h, C.byref(pref), C.byref(mini)))
        return int(pref.value), int(mini.value)

    def numeric(self, row_ptr=None, out=None, host_out=None, workspace=None):
        """magnus_numeric (reference magnus.py:459-542): fills C; returns (C, counters).
        host_out=(col, val): host tensors (page-locked for overlap) that receive C's col / val;
        completed row ranges are read back while later row batches compute.
        workspace: a caller-owned device tensor (>= workspace_bytes()[1] bytes) that holds the
        heavy rows' reorder buffer instead of the library's pool."""
        if workspace is not None:
            if not workspace.is_cuda:
                raise InputError("workspace must be a device tensor")
            nbytes = workspace.numel() * workspace.element_size()
            _lib.check(_lib.lib().magnus_set_workspace(self.ctx.h, C.c_void_p(workspace.data_ptr()), C.c_int64(nbytes)))
        try:
            return self._numeric(row_ptr, out, host_out)
        finally:
            if workspace is not None:
                _lib.lib().magnus_set_workspace(self.ctx.h, None, C.c_int64(0))

    def _numeric(self, row_ptr=None, out=None, host_out=None):
        torch = _torch()
        rp = self.row_ptr if row_ptr is None else row_ptr
        if rp is None or rp is not self.row_ptr:
            raise ContractViolation("row_ptr does not come from a symbolic pass of (A, B)")
        if out is None:
            col = torch.empty(self.nnz, dtype=torch.int32, device=self.device)
            val = torch.empty(self.nnz, dtype=torch.float64, device=self.device)
        else:
            col, val = out
        cnt = _lib.Counters()
        if host_out is None:
            _lib.check(_lib.lib().magnus_numeric(self.ctx.h, C.c_void_p(rp.data_ptr()), C.c_void_p(col.data_ptr()),
                                                 C.c_void_p(val.data_ptr()), C.byref(cnt),
                                                 C.c_void_p(self.stream.cuda_stream)))
        else:
            hc, hv = host_out
            if hc.numel() < self.nnz or hv.numel() < self.nnz or hc.is_cuda or hv.is_cuda:
                raise InputError("host_out buffers must be host tensors with at least nnz(C) entries")
            _lib.check(_lib.lib().magnus_numeric_host(self.ctx.h, C.c_void_p(rp.data_ptr()), C.c_void_p(col.data_ptr()),
                                                      C.c_void_p(val.data_ptr()), C.c_void_p(hc.data_ptr()),
                                                      C.c_void_p(hv.data_ptr()), C.byref(cnt),
                                                      C.c_void_p(self.stream.cuda_stream)))
        counters = {n: int(getattr(cnt, n)) for n, _ in _lib.Counters._fields_}
        return CsrMatrix(self.A.n_rows, self.B.n_cols, rp, col, val, canonical=True), counters

    def launches(self) -> int:
        return self.ctx.launches()

    def close(self):
        self.ctx.close()


def spgemm_magnus(A: CsrMatrix, B: CsrMatrix, sys: SystemParams = None, thresholds: AccumThresholds = None,
                  threads: int = 1, force_fine_only: bool = False) -> SpgemmResult:
    """Full pipeline: stats, plans, categorization, symbolic, numeric (reference magnus.py:545-583)."""
    _check_dims(A, B)
    torch = _torch()
    t0 = time.perf_counter()
    plan = MagnusPlan(A, B, sys, thresholds, force_fine_only)
    plan.stream.synchronize()
    t1 = time.perf_counter()
    rp = plan.symbolic()
    t2 = time.perf_counter()
    Cd, counters = plan.numeric(rp)
    plan.stream.synchronize()
    t3 = time.perf_counter()
    Cm = Cd
    if plan.host_io:
        col = Cd.col.cpu().numpy().view(np.uint32)
        Cm = CsrMatrix(Cd.n_rows, Cd.n_cols, Cd.row_ptr.cpu().numpy(), col, Cd.val.cpu().numpy(), canonical=True)
    t4 = time.perf_counter()
    plan.close()
    del torch
    return SpgemmResult(Cm, {"setup": t1 - t0, "symbolic": t2 - t1, "numeric": t3 - t2, "post": t4 - t3}, counters)


def row_intermediate_stats(A: CsrMatrix, B: CsrMatrix) -> RowStats:
    """Reference gustavson.py:97-134 on the device (torch int64 tensors)."""
    torch = _torch()
    _check_dims(A, B)
    dev = torch.device("cuda", torch.cuda.current_device())
    dA = _to_device(A, dev)
    dB = dA if B is A else _to_device(B, dev)
    n = A.n_rows
    inter = torch.empty(n, dtype=torch.int64, device=dev)
    mn = torch.empty(n, dtype=torch.int64, device=dev)
    mx = torch.empty(n, dtype=torch.int64, device=dev)
    a, b = _abi(dA), _abi(dB)
    _lib.check(_lib.lib().magnus_row_stats(C.byref(a), C.byref(b), C.c_void_p(inter.data_ptr()), C.c_void_p(mn.data_ptr()),
                                           C.c_void_p(mx.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return RowStats(inter, mn, mx)


def categorize_rows(stats: RowStats, plan, sys: SystemParams, thresholds: AccumThresholds) -> RowCategories:
    """Reference magnus.py:68-94 (first matching rule wins): Sort if inter < crossover, Dense if
    the row's column window fits l2 at the numeric cost (val_bytes + 1 per column), else Fine --
    or Coarse for every such row when the plan uses the coarse level.  Works on numpy arrays and
    on torch tensors (device-resident stats from `row_intermediate_stats` stay on the device);
    the device pipeline applies the same rule in k_categorize."""
    inter, rng = stats.inter_size, stats.range_len
    is_sort = inter < thresholds.sort_dense_crossover
    is_dense = ~is_sort & (rng * (sys.val_bytes + 1) <= sys.l2_bytes)
    rest = ~is_sort & ~is_dense
    none = is_sort & ~is_sort
    is_fine, is_coarse = (none, rest) if plan.use_coarse else (rest, none)
    if isinstance(inter, np.ndarray):
        idx = np.flatnonzero
    else:
        def idx(m):
            return _torch().nonzero(m).flatten()
    return RowCategories(idx(is_sort), idx(is_dense), idx(is_fine), idx(is_coarse))


# The two phases as separate calls with the reference's signatures (magnus.py:420, 459).  The
# device keeps per-row chunk tables between them; a numeric call reuses the plan of the symbolic
# call that produced its row_ptr, and otherwise runs the symbolic pass itself first.
_LAST_PLAN = {}


def _force_fine_from(plan, sys, n_cols) -> bool:
    full = compute_chunk_plan(sys, max(n_cols, 1), SYMBOLIC, allow_coarse=True)
    return bool(full.use_coarse and not plan.use_coarse)


def magnus_symbolic(A, B, plan, cats, stats, sys, thresholds, threads: int = 1):
    """Reference magnus_symbolic (magnus.py:420-456): the exact C.row_ptr (int64; numpy for host
    inputs, a device tensor for device inputs).  `plan` is the symbolic ChunkPlan (its use_coarse
    selects force_fine_only); categories and stats are recomputed on the device by the same rules
    (`cats`/`stats` are accepted for API compatibility); `threads` is host-side only."""
    _check_dims(A, B)
    thresholds = thresholds if thresholds is not None else AccumThresholds()
    mp = MagnusPlan(A, B, sys, thresholds, force_fine_only=_force_fine_from(plan, sys, B.n_cols))
    rp = mp.symbolic()
    out = rp.cpu().numpy() if mp.host_io else rp
    _LAST_PLAN.clear()
    _LAST_PLAN[id(out)] = (mp, rp, out)
    return out


def magnus_numeric(A, B, row_ptr, plan, cats, stats, sys, thresholds, threads: int = 1) -> SpgemmResult:
    """Reference magnus_numeric (magnus.py:459-542): fills C for a row_ptr from magnus_symbolic;
    ContractViolation if row_ptr is not the symbolic pass's result for (A, B)."""
    _check_dims(A, B)
    n = A.n_rows
    shape = tuple(row_ptr.shape)
    if shape != (n + 1,) or int(row_ptr[0]) != 0:
        raise ContractViolation("row_ptr does not come from a symbolic pass of (A, B)")
    thresholds = thresholds if thresholds is not None else AccumThresholds()
    hit = _LAST_PLAN.pop(id(row_ptr), None)
    t0 = time.perf_counter()
    if hit is not None and hit[2] is row_ptr:
        mp, rp = hit[0], hit[1]
    else:
        # plan is the numeric ChunkPlan here; coarse use is decided the same way
        mp = MagnusPlan(A, B, sys, thresholds, force_fine_only=_force_fine_from(plan, sys, B.n_cols))
        rp = mp.symbolic()
        mine = rp.cpu().numpy() if mp.host_io else rp
        same = np.array_equal(mine, np.asarray(row_ptr)) if mp.host_io else bool((mine == row_ptr.to(mine.device)).all())
        if not same:
            mp.close()
            raise ContractViolation("row_ptr does not come from a symbolic pass of (A, B)")
    Cd, counters = mp.numeric(rp)
    mp.stream.synchronize()
    t1 = time.perf_counter()
    Cm = Cd
    if mp.host_io:
        Cm = CsrMatrix(Cd.n_rows, Cd.n_cols, np.asarray(row_ptr), Cd.col.cpu().numpy().view(np.uint32),
                       Cd.val.cpu().numpy(), canonical=True)
    mp.close()
    return SpgemmResult(Cm, {"numeric": t1 - t0}, counters)
