import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from paper_2501_07056_b200 import _lib
if os.environ.get("PHASE_LIB"):
    _lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import AccumThresholds, SystemParams, generate, spgemm_magnus
B200 = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 31)
FINE4K = SystemParams(cache_line_bytes=64, l2_bytes=4096)
th = AccumThresholds(sort_dense_crossover=1024, sort_sweet_spot=8)
A = generate.rmat(14, 16, seed=31)
for name, sp in (("b200", B200), ("fine4k", FINE4K)):
    print(name, flush=True)
    r = spgemm_magnus(A, A, sys=sp, thresholds=th)
    print("ok", r.C.nnz, flush=True)
