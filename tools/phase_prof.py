"""Debug: per-phase cycle breakdown of k_heavy_numeric (builds a -DMG_PROFILE_PHASES copy of the library)."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
from paper_2501_07056_b200 import _lib  # noqa: E402

so = os.path.join(ROOT, "paper_2501_07056_b200", "libmagnus_b200_phases.so")
if len(sys.argv) > 2 and sys.argv[2] == "build":
    cus = [p for p in _lib.sources() if p.endswith(".cu")]
    subprocess.check_call(["nvcc", *_lib.NVCC_FLAGS, "-DMG_PROFILE_PHASES", "-o", so, *cus])
    sys.exit(0)
_lib.LIB_PATH = so
import torch  # noqa: E402
from paper_2501_07056_b200 import MagnusPlan, detect_device_params, generate  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A, B = generate.make_config_device(cfg, rp_dtype=torch.int32)
L = _lib.lib()
L.magnus_debug_phases.argtypes = [C.c_void_p, C.c_int]
out = (C.c_ulonglong * 16)()
plan = MagnusPlan(A, B, sys=detect_device_params())
plan.ctx.profile(True)
rp = plan.symbolic()
L.magnus_debug_phases(out, 1)
Cm, _ = plan.numeric(rp)
print(plan.ctx.profile_read())
L.magnus_debug_phases(out, 1)
names = ["choose window", "wide stage+mark", "wide rank", "wide elect", "dense stage", "dense sort", "dense reduce",
         "dense emit", "advance", "row load", "#windows", "#dense batches", "#rows nk>512", "#segment passes",
         "#elements", "wide reduce"]
timers = [0, 1, 2, 3, 15, 4, 5, 6, 7, 8, 9]
tot = sum(out[i] for i in timers)
for i in timers + [10, 11, 12, 13, 14]:
    v = out[i]
    print(f"{names[i]:>16}: {v:>16d}" + (f"  {100.0 * v / max(tot, 1):5.1f}%" if i in timers else ""))
