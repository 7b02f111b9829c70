"""Golden vectors for the Gustavson baselines, from the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_gustavson.py

For every input case of golden_v1.npz it runs the reference's
`gustavson_dense` and `gustavson_esc` (gustavson.py:253-268) and records
their C as differences against the MAGNUS C already stored in golden_v1
(same pattern, asserted; values stored where their bits differ) plus the
counters.  Output: tests/golden/golden_gustavson_v1.npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..")))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from spgemm.gustavson import gustavson_dense, gustavson_esc  # noqa: E402  (reference package)
from spgemm.matrix import CsrMatrix as RefCsr  # noqa: E402

import golden_util as gu  # noqa: E402

OUT = os.path.join(HERE, "golden_gustavson_v1.npz")


def ref_csr(m):
    return RefCsr(m.n_rows, m.n_cols, np.asarray(m.row_ptr, np.int64), np.asarray(m.col).astype(np.uint32),
                  np.asarray(m.val, np.float64))


def main():
    arrays, man = gu.load()
    out, cases = {}, []
    seen = set()
    for rec in man["cases"]:
        case = rec["case"]
        if "shape" not in rec or case in seen:
            continue
        seen.add(case)
        A, B = gu.inputs(case)
        rA = ref_csr(A)
        rB = rA if B is A else ref_csr(B)
        base_rp, base_col = arrays[f"{case}/base/C_rp"], arrays[f"{case}/base/C_col"]
        base_val = arrays[f"{case}/base/C_val"]
        entry = {"case": case}
        for algo, fn in (("dense", gustavson_dense), ("esc", gustavson_esc)):
            r = fn(rA, rB, threads=1)
            C = r.C
            assert np.array_equal(np.asarray(C.row_ptr, np.int64), base_rp), case
            assert np.array_equal(np.asarray(C.col).astype(np.uint32), base_col), case
            val = np.asarray(C.val, np.float64)
            d = np.nonzero(val.view(np.uint64) != base_val.view(np.uint64))[0]
            out[f"{case}/{algo}/diff_idx"] = d.astype(np.int64)
            out[f"{case}/{algo}/diff_val"] = val[d]
            entry[algo] = {"counters": {k: int(v) for k, v in r.counters.items()}, "n_diff": int(d.size)}
        cases.append(entry)
        print(case, entry["dense"]["n_diff"], entry["esc"]["n_diff"])
    out["manifest"] = np.frombuffer(json.dumps({"cases": cases}).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
