"""Generate golden vectors by running the UNMODIFIED reference implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `spgemm.magnus.spgemm_magnus` (reference magnus.py:545-583) and
records, for a corpus of small inputs and a sweep of SystemParams (forced
sort / dense / fine / coarse categorisation, multi-batch coarse, force-fine-only,
an over-budget row -- SPEC.md:452-453), the reference's C (row_ptr, col, val bits)
and counters.  The fixtures are committed as tests/golden/golden_v1.npz and pin
both the CPU oracle (oracle/) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from spgemm.errors import OverBudgetError  # noqa: E402  (reference package)
from spgemm.magnus import spgemm_magnus  # noqa: E402
from spgemm.matrix import CsrMatrix as RefCsr  # noqa: E402
from spgemm.planner import SystemParams as RefSys  # noqa: E402

from paper_2501_07056_b200 import generate as G  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "golden_v1.npz")

SYSTEMS = {
    "host2m": dict(cache_line_bytes=64, l2_bytes=2 << 20, memory_budget_bytes=1 << 31),
    "b200": dict(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 31),
    "mid64k": dict(cache_line_bytes=64, l2_bytes=65536, memory_budget_bytes=1 << 31),
    "fine4k": dict(cache_line_bytes=64, l2_bytes=4096, memory_budget_bytes=1 << 31),
    "coarse512": dict(cache_line_bytes=64, l2_bytes=512, memory_budget_bytes=1 << 31),
    "coarse700": dict(cache_line_bytes=64, l2_bytes=700, memory_budget_bytes=1 << 31),
    "coarse700_budget": dict(cache_line_bytes=64, l2_bytes=700, memory_budget_bytes=12 * 6000),
}


def ref_csr(m):
    return RefCsr(m.n_rows, m.n_cols, np.asarray(m.row_ptr, np.int64), np.asarray(m.col).astype(np.uint32),
                  np.asarray(m.val, np.float64))


def random_csr(rng, n, m, density, integer):
    mask = rng.random((n, m)) < density
    vals = rng.integers(-3, 4, size=(n, m)).astype(np.float64) if integer else rng.uniform(-1, 1, size=(n, m))
    vals[vals == 0] = 1.0
    rows, cols = np.nonzero(mask)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return G.CsrMatrix(n, m, rp, cols.astype(np.int32), vals[rows, cols])


def hub_case():
    """One A row with 200 nonzeros whose B rows all hit column 5: a 200-term
    sort-mode segment (numpy pairwise recursion branch), plus mixed rows."""
    n = 256
    rng = np.random.default_rng(7)
    a_rows = [np.arange(200)] + [np.sort(rng.choice(n, size=rng.integers(0, 40), replace=False)) for _ in range(n - 1)]
    b_rows = []
    for k in range(n):
        extra = rng.choice(np.arange(6, n), size=rng.integers(0, 3), replace=False) if k % 3 else np.array([], int)
        b_rows.append(np.sort(np.r_[5, extra]).astype(np.int64))

    def build(rowlist, vals_seed):
        rp = np.zeros(len(rowlist) + 1, np.int64)
        np.cumsum([len(r) for r in rowlist], out=rp[1:])
        col = np.concatenate(rowlist).astype(np.int32)
        val = np.random.default_rng(vals_seed).uniform(-1, 1, col.size)
        return G.CsrMatrix(len(rowlist), n, rp, col, val)

    return build(a_rows, 1), build(b_rows, 2)


def corpus():
    rng = np.random.default_rng(2501_07056)
    cases = []
    for t in range(24):
        n, k, m = (int(x) for x in rng.integers(1, 129, size=3))
        dens = float(rng.choice([0.0, 0.01, 0.05, 0.2, 0.6, 1.0]))
        integer = bool(t % 2)
        A = random_csr(rng, n, k, dens, integer)
        B = random_csr(rng, k, m, float(rng.choice([0.05, 0.2, 0.6, 1.0])), integer)
        cases.append((f"rand{t}", A, B, ["host2m", "fine4k", "coarse512"]))
    R = G.rmat(10, 8, seed=11)
    cases.append(("rmat10", R, R, list(SYSTEMS)))
    R9 = G.rmat(9, 8, seed=12)
    cases.append(("rmat9", R9, R9, ["host2m", "fine4k", "coarse512", "coarse700", "coarse700_budget"]))
    S = G.stencil27(6)
    cases.append(("stencil6", S, S, ["host2m", "b200", "fine4k", "coarse512"]))
    U = G.uniform_rows(2048, 2048, 16, seed=13)
    cases.append(("uniform2k", U, U, ["host2m", "b200", "fine4k"]))
    U1 = G.uniform_rows(2048, 16384, 8, seed=14)
    U2 = G.uniform_rows(16384, 1 << 18, 8, seed=15)
    cases.append(("uniformAB", U1, U2, ["host2m", "b200", "fine4k", "coarse512"]))
    H = hub_case()
    cases.append(("hub", H[0], H[1], ["host2m", "b200", "fine4k", "coarse512"]))
    E = G.CsrMatrix(5, 7, np.zeros(6, np.int64), np.empty(0, np.int32), np.empty(0))
    F = random_csr(rng, 7, 3, 0.5, True)
    cases.append(("emptyA", E, F, ["host2m"]))
    I4 = G.CsrMatrix(4, 4, np.arange(5, dtype=np.int64), np.arange(4, dtype=np.int32), np.ones(4))
    cases.append(("identity4", I4, I4, ["host2m", "coarse512"]))
    return cases


def main():
    arrays = {}
    manifest = []
    for name, A, B, systems in corpus():
        arrays[f"{name}/A_rp"] = np.asarray(A.row_ptr, np.int64)
        arrays[f"{name}/A_col"] = np.asarray(A.col, np.int32)
        arrays[f"{name}/A_val"] = np.asarray(A.val, np.float64)
        same = A is B
        if not same:
            arrays[f"{name}/B_rp"] = np.asarray(B.row_ptr, np.int64)
            arrays[f"{name}/B_col"] = np.asarray(B.col, np.int32)
            arrays[f"{name}/B_val"] = np.asarray(B.val, np.float64)
        for sname in systems:
            for ffo in ([False, True] if sname == "coarse512" and name.startswith("rmat") else [False]):
                sysp = RefSys(**SYSTEMS[sname])
                key = f"{name}/{sname}/{int(ffo)}"
                rec = dict(case=name, sys=sname, force_fine_only=ffo, shape=[A.n_rows, A.n_cols, B.n_cols],
                           same=same)
                try:
                    res = spgemm_magnus(ref_csr(A), ref_csr(B), sys=sysp, threads=1, force_fine_only=ffo)
                except OverBudgetError as e:
                    rec["error"] = "OverBudgetError"
                    rec["message"] = str(e)
                    manifest.append(rec)
                    continue
                base = f"{name}/base"
                if f"{base}/C_rp" not in arrays:
                    arrays[f"{base}/C_rp"] = res.C.row_ptr.astype(np.int64)
                    arrays[f"{base}/C_col"] = res.C.col.astype(np.uint32)
                    arrays[f"{base}/C_val"] = res.C.val.astype(np.float64)
                    rec["base"] = True
                else:
                    assert np.array_equal(arrays[f"{base}/C_rp"], res.C.row_ptr)
                    assert np.array_equal(arrays[f"{base}/C_col"], res.C.col)
                    diff = np.flatnonzero(arrays[f"{base}/C_val"].view(np.uint64) != res.C.val.view(np.uint64))
                    arrays[f"{key}/diff_idx"] = diff.astype(np.int64)
                    arrays[f"{key}/diff_val"] = res.C.val[diff].astype(np.float64)
                    rec["n_diff_vs_base"] = int(diff.size)
                rec["counters"] = {k: int(v) for k, v in res.counters.items()}
                manifest.append(rec)
                print(key, rec["counters"])
    # an over-budget case: a single coarse row larger than the budget
    R = G.rmat(9, 8, seed=12)
    sysp = RefSys(cache_line_bytes=64, l2_bytes=512, memory_budget_bytes=64)
    try:
        spgemm_magnus(ref_csr(R), ref_csr(R), sys=sysp, threads=1)
        manifest.append(dict(case="rmat9", sys="overbudget", error=None))
    except OverBudgetError as e:
        manifest.append(dict(case="rmat9", sys="overbudget", force_fine_only=False, error="OverBudgetError",
                             message=str(e), sysdict=dict(cache_line_bytes=64, l2_bytes=512, memory_budget_bytes=64)))
    arrays["manifest"] = np.frombuffer(json.dumps(dict(systems=SYSTEMS, cases=manifest)).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
