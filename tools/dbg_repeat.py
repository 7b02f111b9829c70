"""Debug: repeat symbolic (+ numeric) on one R-MAT and check run-to-run determinism."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2501_07056_b200 import _lib  # noqa: E402
if os.environ.get("PHASE_LIB"):
    _lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import MagnusPlan, SystemParams, generate  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 15
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
A = generate.rmat_device(scale, 16, seed=7)
sysp = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 30)
if len(sys.argv) > 2 and sys.argv[2] == "small":
    sysp = SystemParams(cache_line_bytes=64, l2_bytes=16384)
ref = None
for path in ("binned", "direct"):
    os.environ["MAGNUS_HEAVY_PATH"] = path
    for r in range(reps):
        plan = MagnusPlan(A, A, sys=sysp)
        rp = plan.symbolic()
        if ref is None:
            ref = rp.clone()
        same = bool(torch.equal(rp, ref))
        try:
            C, cnt = plan.numeric(rp)
            st = "ok"
        except Exception as ex:
            st = type(ex).__name__
        plan.close()
        bad = (rp != ref).nonzero().flatten()[:5].tolist()
        print(path, r, "row_ptr same:", same, bad, "numeric:", st, flush=True)
