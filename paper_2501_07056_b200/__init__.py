"""B200-native MAGNUS SpGEMM (C = A.B, CSR in, CSR out) -- drop-in for the
reference package's `spgemm_magnus` (arxiv/paper_2501_07056, magnus.py:545-583).

Public API (same names as the reference):
    spgemm_magnus, CsrMatrix, RowStats, SystemParams, ChunkPlan, compute_chunk_plan,
    with_overrides, AccumThresholds, select_accumulator, merge_chunks_for_sort,
    SpgemmResult, RowCategories, row_intermediate_stats, IdealBoundInputs / ideal_bound /
    bound_inputs_for (the paper's minimum-data-volume model) and the error classes.
Device-only additions: detect_device_params, MagnusPlan (the two phases),
parallel.spgemm_magnus_distributed (row-block split over ranks).
Baselines (reference gustavson.py:155-268, on the device): gustavson_dense, gustavson_esc and their phases.
"""

from .accumulators import Accum, AccumThresholds, merge_chunks_for_sort, select_accumulator
from .bound import IdealBoundInputs, bound_inputs_for, col_index_bytes, ideal_bound
from .errors import ContractViolation, InputError, OverBudgetError, ParseError, SpgemmError
from .matrix import (CscSubMatrix, CsrMatrix, RowStats, ValidationReport, canonicalize_csr, check_csr, csr_from_arrays,
                     csr_from_triplets, csr_rows_to_csc, validate_csr)
from .planner import (NUMERIC, SYMBOLIC, ChunkPlan, SystemParams, b200_default_params, compute_chunk_plan,
                      detect_device_params, with_overrides)

__all__ = [
    "Accum", "AccumThresholds", "merge_chunks_for_sort", "select_accumulator", "ContractViolation", "InputError",
    "OverBudgetError", "ParseError", "SpgemmError", "CsrMatrix", "RowStats", "validate_csr", "NUMERIC", "SYMBOLIC",
    "ChunkPlan", "SystemParams", "b200_default_params", "compute_chunk_plan", "detect_device_params", "with_overrides",
    "spgemm_magnus", "SpgemmResult", "RowCategories", "MagnusPlan", "row_intermediate_stats", "IdealBoundInputs",
    "bound_inputs_for", "col_index_bytes", "ideal_bound", "gustavson_dense", "gustavson_esc", "gustavson_dense_symbolic",
    "gustavson_dense_numeric", "gustavson_esc_numeric", "categorize_rows", "magnus_symbolic", "magnus_numeric",
    "CscSubMatrix", "ValidationReport", "canonicalize_csr", "check_csr", "csr_from_arrays", "csr_from_triplets",
    "csr_rows_to_csc", "release_workspace",
]


_GUSTAVSON = ("gustavson_dense", "gustavson_esc", "gustavson_dense_symbolic", "gustavson_dense_numeric",
              "gustavson_esc_numeric")


def __getattr__(name):
    # the CUDA-backed entry points load the extension lazily (importing the
    # package must not need a GPU); a missing extension raises ImportError.
    if name in ("spgemm_magnus", "SpgemmResult", "RowCategories", "MagnusPlan", "row_intermediate_stats",
                "categorize_rows", "magnus_symbolic", "magnus_numeric"):
        from . import magnus
        return getattr(magnus, name)
    if name == "release_workspace":
        from . import _lib
        return _lib.release_workspace
    if name in _GUSTAVSON:
        from . import gustavson
        return getattr(gustavson, name)
    raise AttributeError(name)
