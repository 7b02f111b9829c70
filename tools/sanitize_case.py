"""Small products that reach every device kernel class (warp / CTA / dense rows, heavy symbolic,
expand, big-chunk and small-chunk reducers, the direct and fused big-chunk kernels, the coarse
level, fused rows), for
compute-sanitizer (memcheck / racecheck / synccheck).  Checks the result against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2501_07056_b200 import SystemParams, generate, spgemm_magnus  # noqa: E402

B200 = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 31)
FINE4K = SystemParams(cache_line_bytes=64, l2_bytes=4096)
COARSE = SystemParams(cache_line_bytes=64, l2_bytes=1400)   # Coarse-category rows: the device coarse level
cases = [("rmat12", generate.rmat(12, 16, seed=3)), ("stencil", generate.stencil27(10))]
for name, A in cases:
    for sname, sysp in (("b200", B200), ("fine4k", FINE4K), ("coarse", COARSE)):
        ref = oracle.spgemm(A, A, sysp)
        for mode in ("", "direct", "fused"):
            if mode:
                os.environ["MAGNUS_BIG_PATH"] = mode
            else:
                os.environ.pop("MAGNUS_BIG_PATH", None)
            res = spgemm_magnus(A, A, sys=sysp)
            ok = np.array_equal(res.C.col, ref.col) and np.array_equal(res.C.val.view(np.uint64), ref.val.view(np.uint64))
            print(name, sname, mode or "binned", "OK" if ok else "MISMATCH", flush=True)
            assert ok
