"""Loader for tests/golden/golden_gustavson_v1.npz (reference gustavson_dense /
gustavson_esc outputs, stored as bit differences against golden_v1's C)."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

import golden_util as gu

PATH = os.path.join(os.path.dirname(__file__), "golden", "golden_gustavson_v1.npz")


@lru_cache(maxsize=1)
def load():
    z = np.load(PATH)
    arrays = {k: z[k] for k in z.files}
    man = json.loads(bytes(arrays.pop("manifest")).decode())
    return arrays, man


def cases():
    return [c["case"] for c in load()[1]["cases"]]


def expected(case: str, algo: str):
    """(row_ptr, col, val, counters) of the reference's gustavson_<algo> on the case's inputs."""
    a, man = load()
    g, _ = gu.load()
    rp = g[f"{case}/base/C_rp"]
    col = g[f"{case}/base/C_col"]
    val = g[f"{case}/base/C_val"].copy()
    val[a[f"{case}/{algo}/diff_idx"]] = a[f"{case}/{algo}/diff_val"]
    rec = next(c for c in man["cases"] if c["case"] == case)
    return rp, col, val, rec[algo]["counters"]
