"""Loader for tests/golden/golden_v1.npz (made by tests/golden/make_golden.py
from the unmodified reference).  Reconstructs inputs and the reference's C."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

from paper_2501_07056_b200.matrix import CsrMatrix
from paper_2501_07056_b200.planner import SystemParams

PATH = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@lru_cache(maxsize=1)
def load():
    z = np.load(PATH)
    arrays = {k: z[k] for k in z.files}
    manifest = json.loads(bytes(arrays.pop("manifest")).decode())
    return arrays, manifest


def inputs(case: str):
    a, man = load()
    rec = next(c for c in man["cases"] if c["case"] == case and "shape" in c)
    n, k, m = rec["shape"]
    A = CsrMatrix(n, k, a[f"{case}/A_rp"], a[f"{case}/A_col"], a[f"{case}/A_val"])
    if f"{case}/B_rp" in a:
        B = CsrMatrix(k, m, a[f"{case}/B_rp"], a[f"{case}/B_col"], a[f"{case}/B_val"])
    else:
        B = A
    return A, B


def system(name: str, rec=None) -> SystemParams:
    _, man = load()
    if rec is not None and "sysdict" in rec:
        return SystemParams(**rec["sysdict"])
    return SystemParams(**man["systems"][name])


def expected(rec):
    """(row_ptr, col uint32, val float64) of the reference run described by rec."""
    a, _ = load()
    case = rec["case"]
    rp = a[f"{case}/base/C_rp"]
    col = a[f"{case}/base/C_col"]
    val = a[f"{case}/base/C_val"].copy()
    key = f"{case}/{rec['sys']}/{int(rec['force_fine_only'])}"
    if f"{key}/diff_idx" in a:
        val[a[f"{key}/diff_idx"]] = a[f"{key}/diff_val"]
    return rp, col, val


def runs():
    """Every reference run in the manifest (including expected errors)."""
    _, man = load()
    return man["cases"]
