"""Debug: wave/conflict statistics of the big-chunk reducer (build with -DMG_BIG_STATS via tools/variants.py)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import MagnusPlan, detect_device_params, generate  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "3"
if arg.startswith("rmat"):   # rmatSCALE: a smaller R-MAT, ef 16
    A = B = generate.rmat_device(int(arg[4:]), 16, seed=3, rp_dtype=torch.int32)
else:
    A, B = generate.make_config_device(int(arg), rp_dtype=torch.int32)
plan = MagnusPlan(A, B, sys=detect_device_params())
rp = plan.symbolic()
Cm, _ = plan.numeric(rp)
torch.cuda.synchronize()
L = _lib.lib()
out = (C.c_ulonglong * 8)()
L.magnus_debug_big_stats.argtypes = [C.c_void_p]
L.magnus_debug_big_stats(out)
waves, brk, maxg, lanes = out[0], out[1], out[2], out[3]
tm, ta, te = out[4], out[5], out[6]
tt = max(tm + ta + te, 1)
print(f"cycles: mark+prefix {100 * tm / tt:.1f}%  accumulate {100 * ta / tt:.1f}%  emit {100 * te / tt:.1f}%  "
      f"accumulate cycles/wave {ta / max(waves, 1):.0f}")
print(f"waves {waves} lanes/wave {lanes / max(waves, 1):.1f} waves-with-repeats {brk} ({100 * brk / max(waves, 1):.1f}%) "
      f"mean maxg {maxg / max(brk, 1):.2f}")
