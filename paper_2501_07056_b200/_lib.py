"""ctypes binding of the C-ABI in include/magnus_b200.h (libmagnus_b200.so).

The shared library is built in-tree for sm_100a by `build()` (nvcc) and is the
only compute path: there is no CPU fallback.  Loading fails loudly if it is
missing.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

from .errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libmagnus_b200.so")
CSRC = os.path.join(HERE, "csrc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into libmagnus_b200.so (sm_100a).  No GPU needed."""
    srcs = sources()
    hdrs = [os.path.join(ROOT, "include", h) for h in ("magnus_b200.h", "magnus_gen.h")]
    newest = max(os.path.getmtime(p) for p in srcs + hdrs)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    cus = [p for p in srcs if p.endswith(".cu")]
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB_PATH + ".tmp", *cus]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p),
                ("rp_bytes", C.c_int32), ("col", C.c_void_p), ("val", C.c_void_p)]


class Sys(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("cache_line_bytes", "l2_bytes", "memory_budget_bytes", "histo_type_bytes",
                                         "prefix_sum_type_bytes", "val_bytes")]


class Thresholds(C.Structure):
    _fields_ = [("sort_dense_crossover", C.c_int64), ("sort_sweet_spot", C.c_int64)]


class Plan(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("plan_cols", "s_dense_accum", "s_chunk_fine", "n_chunks_fine", "chunk_len_fine",
                                         "shift_fine", "m_max_l2", "use_coarse", "n_chunks_coarse", "chunk_len_coarse",
                                         "shift_coarse")]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("nnz_c", "inter_prod_size", "coarse_batches", "rows_sort", "rows_dense",
                                         "rows_fine", "rows_coarse")]


# every symbol include/magnus_b200.h declares
EXPORTS = ["magnus_compute_chunk_plan", "magnus_ctx_create", "magnus_ctx_destroy", "magnus_setup", "magnus_symbolic",
           "magnus_numeric", "magnus_row_stats", "magnus_categories", "magnus_launch_count", "magnus_last_error",
           "magnus_version", "magnus_profile_enable", "magnus_profile_read", "magnus_heavy_stats",
           "magnus_numeric_host", "magnus_gd_scratch_bytes", "magnus_gd_symbolic", "magnus_gd_numeric",
           "magnus_esc_expand", "magnus_esc_compress", "magnus_mb_histogram", "magnus_mb_reorder_scratch_bytes",
           "magnus_mb_reorder", "magnus_mb_dense", "magnus_mb_stream",
           "magnus_mb_scan_scratch_bytes", "magnus_mb_scan", "magnus_release_workspace", "magnus_workspace_reserved", "magnus_workspace_bytes", "magnus_set_workspace",
           "magnus_coarse_level_stats", "magnus_sort_pairs_scratch_bytes", "magnus_sort_pairs"]
KERNEL_NAMES = ["row_stats", "categorize", "sym_warp", "sym_block", "sym_heavy", "scan", "num_warp", "num_block",
                "num_heavy", "sym_dense", "num_dense", "bin_plan", "bin_expand", "bin_reduce", "bin_big", "dir_index",
                "dir_plan", "dir_num"]
GEN_EXPORTS = ["magnus_gen_rmat_keys", "magnus_gen_uniform_pm1", "magnus_gen_uniform_rows"]

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.magnus_last_error.restype = C.c_char_p
        L.magnus_version.restype = C.c_char_p
        L.magnus_launch_count.restype = C.c_int64
        L.magnus_launch_count.argtypes = [C.c_void_p]
        L.magnus_ctx_destroy.argtypes = [C.c_void_p]
        L.magnus_ctx_destroy.restype = None
        L.magnus_ctx_create.argtypes = [C.POINTER(C.c_void_p)]
        L.magnus_setup.argtypes = [C.c_void_p, C.POINTER(Csr), C.POINTER(Csr), C.POINTER(Sys), C.POINTER(Thresholds),
                                   C.c_int, C.c_void_p]
        L.magnus_symbolic.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.magnus_numeric.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Counters), C.c_void_p]
        L.magnus_numeric_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.POINTER(Counters), C.c_void_p]
        L.magnus_row_stats.argtypes = [C.POINTER(Csr), C.POINTER(Csr), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_categories.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_gen_rmat_keys.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_double,
                                           C.c_double, C.c_void_p, C.c_void_p]
        L.magnus_gen_uniform_pm1.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]
        L.magnus_gen_uniform_rows.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p]
        L.magnus_profile_enable.argtypes = [C.c_void_p, C.c_int]
        L.magnus_profile_read.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_heavy_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.magnus_coarse_level_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.magnus_sort_pairs_scratch_bytes.restype = C.c_size_t
        L.magnus_sort_pairs_scratch_bytes.argtypes = [C.c_int64]
        L.magnus_sort_pairs.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_compute_chunk_plan.argtypes = [C.POINTER(Sys), C.c_int64, C.c_int, C.c_int, C.POINTER(Plan)]
        L.magnus_gd_scratch_bytes.restype = C.c_size_t
        L.magnus_gd_scratch_bytes.argtypes = [C.c_int64, C.c_int64]
        L.magnus_gd_symbolic.argtypes = [C.POINTER(Csr), C.POINTER(Csr), C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.magnus_gd_numeric.argtypes = [C.POINTER(Csr), C.POINTER(Csr), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_size_t, C.c_void_p]
        L.magnus_esc_expand.argtypes = [C.POINTER(Csr), C.POINTER(Csr), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        L.magnus_esc_compress.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.magnus_mb_histogram.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.magnus_mb_reorder_scratch_bytes.restype = C.c_size_t
        L.magnus_mb_reorder_scratch_bytes.argtypes = [C.c_int64, C.c_int]
        L.magnus_mb_reorder.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_mb_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        L.magnus_mb_scan_scratch_bytes.restype = C.c_size_t
        L.magnus_mb_scan_scratch_bytes.argtypes = [C.c_int64]
        L.magnus_mb_scan.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.magnus_mb_stream.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.magnus_release_workspace.argtypes = []
        L.magnus_workspace_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.magnus_set_workspace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.magnus_workspace_reserved.argtypes = []
        L.magnus_workspace_reserved.restype = C.c_int64
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc:
        raise_for_status(rc, lib().magnus_last_error().decode())


class Context:
    """Owns a magnus_ctx (device workspace between the phases)."""

    def __init__(self):
        h = C.c_void_p()
        check(lib().magnus_ctx_create(C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().magnus_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self) -> int:
        return int(lib().magnus_launch_count(self.h))

    def profile(self, enable: bool = True) -> None:
        check(lib().magnus_profile_enable(self.h, int(enable)))

    def heavy_stats(self) -> dict:
        """Products / distinct columns of heavy rows in big chunks and in the other chunks."""
        out = (C.c_int64 * 4)()
        check(lib().magnus_heavy_stats(self.h, out))
        return {"big_products": int(out[0]), "big_distinct": int(out[1]), "small_products": int(out[2]),
                "small_distinct": int(out[3])}

    def coarse_level_stats(self) -> dict:
        """Rows / batches / CSC entries the device coarse level (Alg. 4) handled in the last numeric call."""
        out = (C.c_int64 * 3)()
        check(lib().magnus_coarse_level_stats(self.h, out))
        return {"rows": int(out[0]), "batches": int(out[1]), "csc_entries": int(out[2])}

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} since the last read (synchronises)."""
        n = len(KERNEL_NAMES)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        check(lib().magnus_profile_read(self.h, ms, cnt))
        return {KERNEL_NAMES[k]: (float(ms[k]), int(cnt[k])) for k in range(n)}


def sort_pairs(keys, key_bits: int = 64, key_mask: int = None):
    """Stable ascending sort of non-negative int64 CUDA keys with the library's own LSD radix sort
    (csrc/radix_sort.cuh): returns (sorted keys, permutation), like torch.sort(keys, stable=True).  The keys may
    differ only in their low `key_bits` bits, or in the bits of `key_mask` (bytes without a set bit cost no pass)."""
    import torch

    n = int(keys.numel())
    out = torch.empty_like(keys)
    perm = torch.empty(n, dtype=torch.int64, device=keys.device)
    if n:
        scratch = torch.empty(int(lib().magnus_sort_pairs_scratch_bytes(n)), dtype=torch.uint8, device=keys.device)
        mask = int(key_mask) if key_mask is not None else (1 << min(int(key_bits), 64)) - 1
        check(lib().magnus_sort_pairs(C.c_void_p(keys.data_ptr()), n, C.c_uint64(mask & 0xFFFFFFFFFFFFFFFF), C.c_void_p(out.data_ptr()),
                                      C.c_void_p(perm.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out, perm


def release_workspace() -> None:
    """Return the library's pooled device workspace to the driver (include/magnus_b200.h)."""
    check(lib().magnus_release_workspace())


def workspace_reserved() -> int:
    """Bytes the library's private workspace pool currently holds on this device."""
    return int(lib().magnus_workspace_reserved())
