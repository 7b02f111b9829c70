"""Debug: small R-MAT through the direct and the binned heavy path; compare bit for bit."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2501_07056_b200 import _lib  # noqa: E402
if os.environ.get("PHASE_LIB"):
    _lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import SystemParams, generate, spgemm_magnus  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 13
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 16
A = generate.rmat(scale, ef, seed=7)
for sysp in (SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 30),
             SystemParams(cache_line_bytes=64, l2_bytes=16384)):
    out = {}
    for path in ("binned", "direct"):
        os.environ["MAGNUS_HEAVY_PATH"] = path
        r = spgemm_magnus(A, A, sys=sysp)
        out[path] = r
        print(path, r.counters, flush=True)
    a, b = out["direct"].C, out["binned"].C
    print("row_ptr", np.array_equal(a.row_ptr, b.row_ptr), "col", np.array_equal(a.col, b.col), "val",
          np.array_equal(a.val.view(np.uint64), b.val.view(np.uint64)))
