"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the C oracle (liboracle.so).

The oracle restates the reference's MAGNUS path on the CPU (see
magnus_oracle.c).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "magnus_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return path


def lib():
    global _LIB
    if _LIB is None:
        _LIB = C.CDLL(build())
        _LIB.oracle_last_error.restype = C.c_char_p
        _LIB.oracle_pairwise_sum.restype = C.c_double
        _LIB.oracle_pairwise_sum.argtypes = [C.c_void_p, C.c_int64]
    return _LIB


class OCsr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p)]


class OSys(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("cache_line_bytes", "l2_bytes", "memory_budget_bytes",
                                         "histo_type_bytes", "prefix_sum_type_bytes", "val_bytes")]


class OThr(C.Structure):
    _fields_ = [("sort_dense_crossover", C.c_int64), ("sort_sweet_spot", C.c_int64)]


class OPlan(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("plan_cols", "s_dense_accum", "s_chunk_fine", "n_chunks_fine", "chunk_len_fine",
                                         "shift_fine", "m_max_l2", "use_coarse", "n_chunks_coarse", "chunk_len_coarse",
                                         "shift_coarse")]


@dataclass
class OracleResult:
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    counters: dict


def _csr(m, keep):
    rp = np.ascontiguousarray(np.asarray(m.row_ptr), dtype=np.int64)
    col = np.ascontiguousarray(np.asarray(m.col)).view(np.uint32) if np.asarray(m.col).dtype.itemsize == 4 else \
        np.ascontiguousarray(np.asarray(m.col).astype(np.uint32))
    val = np.ascontiguousarray(np.asarray(m.val), dtype=np.float64)
    keep.extend([rp, col, val])
    return OCsr(m.n_rows, m.n_cols, rp.ctypes.data, col.ctypes.data, val.ctypes.data)


def _sys(sys):
    return OSys(sys.cache_line_bytes, sys.l2_bytes, sys.memory_budget_bytes, sys.histo_type_bytes,
                sys.prefix_sum_type_bytes, sys.val_bytes)


def _raise(rc):
    from paper_2501_07056_b200.errors import ContractViolation, InputError, OverBudgetError
    msg = lib().oracle_last_error().decode()
    raise {1: InputError, 2: ContractViolation, 3: OverBudgetError}.get(rc, RuntimeError)(msg)


def chunk_plan(sys, m_c: int, numeric: bool, allow_coarse: bool = True) -> dict:
    p = OPlan()
    rc = lib().oracle_compute_chunk_plan(C.byref(_sys(sys)), C.c_int64(m_c), int(numeric), int(allow_coarse), C.byref(p))
    if rc:
        _raise(rc)
    return {n: int(getattr(p, n)) for n, _ in OPlan._fields_}


def setup(A, B, sys, thresholds=None, force_fine_only=False):
    """(inter, min_col, max_col, category) per row -- row_intermediate_stats + categorize_rows."""
    keep = []
    a, b = _csr(A, keep), _csr(B, keep)
    th = OThr(*(thresholds_tuple(thresholds)))
    n = A.n_rows
    inter, mn, mx = (np.empty(n, np.int64) for _ in range(3))
    cat = np.empty(n, np.int8)
    rc = lib().oracle_setup(C.byref(a), C.byref(b), C.byref(_sys(sys)), C.byref(th), int(force_fine_only),
                            inter.ctypes.data_as(C.c_void_p), mn.ctypes.data_as(C.c_void_p),
                            mx.ctypes.data_as(C.c_void_p), cat.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc)
    return inter, mn, mx, cat


def thresholds_tuple(th):
    if th is None:
        return (256, 32)
    return (th.sort_dense_crossover, th.sort_sweet_spot)


def symbolic(A, B, sys, thresholds=None, force_fine_only=False, threads=0):
    """magnus_symbolic only (reference magnus.py:420-456): C.row_ptr (int64, n_rows+1) and the counters."""
    keep = []
    a, b = _csr(A, keep), _csr(B, keep)
    th = OThr(*thresholds_tuple(thresholds))
    rp = np.empty(A.n_rows + 1, np.int64)
    info = np.zeros(7, np.int64)
    rc = lib().oracle_symbolic(C.byref(a), C.byref(b), C.byref(_sys(sys)), C.byref(th), int(force_fine_only),
                               int(threads), rp.ctypes.data_as(C.c_void_p), info.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc)
    return rp


def spgemm(A, B, sys, thresholds=None, force_fine_only=False, threads=0) -> OracleResult:
    """Full reference pipeline (stats, plans, categories, symbolic, numeric) on the CPU."""
    keep = []
    a, b = _csr(A, keep), _csr(B, keep)
    s = _sys(sys)
    th = OThr(*thresholds_tuple(thresholds))
    rp = np.empty(A.n_rows + 1, np.int64)
    info = np.zeros(7, np.int64)
    rc = lib().oracle_symbolic(C.byref(a), C.byref(b), C.byref(s), C.byref(th), int(force_fine_only), int(threads),
                               rp.ctypes.data_as(C.c_void_p), info.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc)
    nnz = int(rp[-1])
    col = np.empty(nnz, np.uint32)
    val = np.empty(nnz, np.float64)
    rc = lib().oracle_numeric(C.byref(a), C.byref(b), C.byref(s), C.byref(th), int(force_fine_only), int(threads),
                              rp.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p),
                              val.ctypes.data_as(C.c_void_p), info.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc)
    keys = ["nnz_c", "inter_prod_size", "coarse_batches", "rows_sort", "rows_dense", "rows_fine", "rows_coarse"]
    return OracleResult(rp, col, val, {k: int(v) for k, v in zip(keys, info)})


def pairwise_sum(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().oracle_pairwise_sum(x.ctypes.data, x.size)


def gustavson(A, B, esc: bool = False, threads: int = 0) -> OracleResult:
    """Reference gustavson_dense / gustavson_esc (gustavson.py:155-268) on the CPU."""
    keep = []
    a, b = _csr(A, keep), _csr(B, keep)
    L = lib()
    rp = np.empty(A.n_rows + 1, np.int64)
    rc = L.oracle_gustavson(C.byref(a), C.byref(b), 0, int(threads), rp.ctypes.data_as(C.c_void_p), None, None)
    if rc:
        _raise(rc)
    nnz = int(rp[-1])
    col = np.empty(nnz, np.uint32)
    val = np.empty(nnz, np.float64)
    rc = L.oracle_gustavson(C.byref(a), C.byref(b), 2 if esc else 1, int(threads), rp.ctypes.data_as(C.c_void_p),
                            col.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p))
    if rc:
        _raise(rc)
    inter = int(np.diff(np.asarray(B.row_ptr).astype(np.int64))[np.asarray(A.col).astype(np.int64)].sum())
    return OracleResult(rp, col, val, {"inter_prod_size": inter, "nnz_c": nnz})
