"""Debug: phases of the host-buffer (e2e) path of bench.py on one config."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_07056_b200 import CsrMatrix, MagnusPlan, detect_device_params, generate  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
A, B = generate.make_config_device(cfg, rp_dtype=torch.int32)
sysp = detect_device_params()
np = bench.np


def pinned(t):
    h = bench.HostBuffer(t.numel(), {torch.int32: np.int32, torch.int64: np.int64, torch.float64: np.float64}[t.dtype])
    h.t.copy_(t)
    return h


bufs = [pinned(t) for t in (A.row_ptr, A.col, A.val)]
Ah = CsrMatrix(A.n_rows, A.n_cols, bufs[0].t, bufs[1].t, bufs[2].t)
Bh = Ah
if B is not A:
    bufs += [pinned(t) for t in (B.row_ptr, B.col, B.val)]
    Bh = CsrMatrix(B.n_rows, B.n_cols, bufs[3].t, bufs[4].t, bufs[5].t)
plan = MagnusPlan(A, B, sys=sysp)
nnz = int(plan.symbolic()[-1])
plan.close()
hc, hv = bench.HostBuffer(nnz, np.int32), bench.HostBuffer(nnz, np.float64)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = MagnusPlan(Ah, Bh, sys=sysp)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rp = plan.symbolic()
    t2 = time.perf_counter()
    C, _ = plan.numeric(rp, host_out=(hc.t, hv.t))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    plan.close()
    del C, rp
    print(f"rep {rep}: plan+H2D {1e3*(t1-t0):.1f} ms  symbolic {1e3*(t2-t1):.1f} ms  numeric+D2H {1e3*(t3-t2):.1f} ms",
          flush=True)
