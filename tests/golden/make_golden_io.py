"""Golden vectors for the matrix-file layer, from the UNMODIFIED reference mmio.py.

Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py

Generates Matrix Market texts procedurally (every field x symmetry, duplicates,
comments, blank lines) and malformed variants, and records what the reference's
read_matrix_market returns (CSR arrays) or raises (ParseError line); the bytes of
its write_binary_cache and the text of its write_matrix_market for two inputs.
Output: tests/golden/io_v1.npz.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..")))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from spgemm import mmio as ref_mmio  # noqa: E402  (reference package)
from spgemm.errors import ParseError as RefParseError  # noqa: E402
from spgemm.matrix import CsrMatrix as RefCsr  # noqa: E402

import golden_util as gu  # noqa: E402

OUT = os.path.join(HERE, "io_v1.npz")


def mm_text(rng, field, sym, n=9, m=7, nnz=20, dup=True):
    if sym != "general":
        m = n
    r = rng.integers(1, n + 1, nnz)
    c = rng.integers(1, m + 1, nnz)
    if sym != "general":
        lo = np.minimum(r, c)
        hi = np.maximum(r, c)
        r, c = hi, lo
        if sym == "skew-symmetric":
            keep = r != c
            r, c = r[keep], c[keep]
    if dup:
        r = np.r_[r, r[:3]]
        c = np.r_[c, c[:3]]
    lines = [f"%%MatrixMarket matrix coordinate {field} {sym}", "% generated", f"{n} {m} {r.size}"]
    for i, (a, b) in enumerate(zip(r, c)):
        v = rng.uniform(-2, 2)
        if field == "pattern":
            lines.append(f"{a} {b}")
        elif field == "integer":
            lines.append(f"{a} {b} {int(rng.integers(-9, 10))}")
        elif field == "complex":
            lines.append(f"{a} {b} {v:.17g} {rng.uniform(-1, 1):.6g}")
        else:
            lines.append(f"{a} {b} {v:.17g}")
        if i == 4:
            lines.append("")
            lines.append("% interleaved comment")
    return "\n".join(lines) + "\n"


def bad_texts():
    good = "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n2 3 4.5\n"
    return {
        "empty": "",
        "banner": "%%MatrixMarket matrix coordinate real\n3 3 0\n",
        "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
        "object": "%%MatrixMarket vector coordinate real general\n3 3 0\n",
        "field": "%%MatrixMarket matrix coordinate double general\n3 3 0\n",
        "symmetry": "%%MatrixMarket matrix coordinate real lower\n3 3 0\n",
        "size_fields": "%%MatrixMarket matrix coordinate real general\n3 3\n",
        "size_int": "%%MatrixMarket matrix coordinate real general\n3 x 1\n1 1 1\n",
        "negative": "%%MatrixMarket matrix coordinate real general\n3 -3 0\n",
        "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
        "too_many": good + "3 3 1.0\n",
        "too_few": good.replace("3 3 2", "3 3 3"),
        "fields": good.replace("2 3 4.5", "2 3"),
        "malformed": good.replace("2 3 4.5", "2 3 4.5x"),
        "out_of_range": good.replace("2 3 4.5", "2 4 4.5"),
        "zero_index": good.replace("1 1 1.0", "0 1 1.0"),
    }


def main():
    rng = np.random.default_rng(2025)
    out, man = {}, {"good": [], "bad": [], "writers": []}
    tmp = tempfile.mkdtemp()
    p = os.path.join(tmp, "m.mtx")
    k = 0
    for field in ("real", "integer", "pattern", "complex"):
        for sym in ("general", "symmetric", "skew-symmetric", "hermitian"):
            for dup in (False, True):
                txt = mm_text(rng, field, sym, dup=dup)
                open(p, "w").write(txt)
                M = ref_mmio.read_matrix_market(p)
                key = f"good{k}"
                out[f"{key}/text"] = np.frombuffer(txt.encode(), np.uint8)
                out[f"{key}/rp"] = np.asarray(M.row_ptr, np.int64)
                out[f"{key}/col"] = np.asarray(M.col).astype(np.uint32)
                out[f"{key}/val"] = np.asarray(M.val, np.float64)
                man["good"].append({"key": key, "shape": [M.n_rows, M.n_cols], "col_dtype": str(M.col.dtype)})
                k += 1
    for name, txt in bad_texts().items():
        open(p, "w").write(txt)
        try:
            ref_mmio.read_matrix_market(p)
            raise SystemExit(f"{name}: reference accepted a malformed file")
        except RefParseError as e:
            out[f"bad_{name}/text"] = np.frombuffer(txt.encode(), np.uint8)
            man["bad"].append({"name": name, "line": e.line})
    for case in ("rmat9", "hub"):
        A, _ = gu.inputs(case)
        R = RefCsr(A.n_rows, A.n_cols, np.asarray(A.row_ptr, np.int64), np.asarray(A.col).astype(np.uint32),
                   np.asarray(A.val, np.float64))
        ref_mmio.write_binary_cache(R, os.path.join(tmp, "a.spgc"))
        ref_mmio.write_matrix_market(R, os.path.join(tmp, "a.mtx"), comment="case " + case)
        out[f"w_{case}/spgc"] = np.fromfile(os.path.join(tmp, "a.spgc"), np.uint8)
        out[f"w_{case}/mtx"] = np.fromfile(os.path.join(tmp, "a.mtx"), np.uint8)
        man["writers"].append({"case": case, "comment": "case " + case})
    out["manifest"] = np.frombuffer(json.dumps(man).encode(), np.uint8)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", len(man["good"]), "good,", len(man["bad"]), "bad")


if __name__ == "__main__":
    main()
