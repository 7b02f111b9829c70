"""Debug: host-side phase times and per-kernel device times of one spgemm call on a BASELINE config."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import _lib  # noqa: E402

if os.environ.get("PHASE_LIB"):   # a variant build (tools/variants.py)
    _lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import MagnusPlan, detect_device_params, generate  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A, B = generate.make_config_device(cfg, rp_dtype=torch.int64 if cfg == 5 else torch.int32)
sysp = detect_device_params()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = MagnusPlan(A, B, sys=sysp)
    plan.ctx.profile(True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rp = plan.symbolic()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    try:
        C, counters = plan.numeric(rp)
    except Exception as ex:   # timing-only variants may break the result
        print("numeric:", type(ex).__name__)
        C = None
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    prof = plan.ctx.profile_read()
    plan.close()
    del C
    print(f"rep {r}: setup {1e3*(t1-t0):.1f} ms  symbolic {1e3*(t2-t1):.1f} ms  numeric {1e3*(t3-t2):.1f} ms  "
          f"total {1e3*(t3-t0):.1f} ms")
    print("   ", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]})
