"""Small workload for ncu captures: C = A.A on a seeded R-MAT (scale, edge factor from argv)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2501_07056_b200 import MagnusPlan, detect_device_params, generate  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 17
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 16
A = generate.rmat_device(scale, ef, seed=3, rp_dtype=torch.int32)
for _ in range(2 if scale < 19 else 1):
    plan = MagnusPlan(A, A, sys=detect_device_params())
    rp = plan.symbolic()
    C, cnt = plan.numeric(rp)
    torch.cuda.synchronize()
    plan.close()
    del C
print("ok", cnt)
