"""Device coarse level (Alg. 4, coarse_rows.cuh) against the fine-level expand on the same Coarse-category rows:
R-MAT 2^scale with SystemParams whose L2 makes the planner choose the coarse level.  Prints step times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2501_07056_b200 import MagnusPlan, SystemParams, compute_chunk_plan, generate  # noqa: E402
from paper_2501_07056_b200.planner import NUMERIC  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
l2 = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
A = generate.rmat_device(scale, 16, seed=5)
sysp = SystemParams(cache_line_bytes=64, l2_bytes=l2, memory_budget_bytes=64 << 30)
pl = compute_chunk_plan(sysp, A.n_cols, NUMERIC)
print("plan: use_coarse", pl.use_coarse, "coarse chunks", pl.n_chunks_coarse, "x", pl.chunk_len_coarse, "fine", pl.chunk_len_fine)
for mode in ("alg4", "fine", "alg4", "fine"):
    if mode == "fine":
        os.environ["MAGNUS_COARSE_PATH"] = "fine"
    else:
        os.environ.pop("MAGNUS_COARSE_PATH", None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = MagnusPlan(A, A, sys=sysp)
    plan.ctx.profile(True)
    rp = plan.symbolic()
    C, counters = plan.numeric(rp)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st = plan.ctx.coarse_level_stats()
    prof = plan.ctx.profile_read()
    plan.close()
    del C
    print(mode, f"{1e3 * (t1 - t0):.1f} ms", "coarse rows", st["rows"], "of", counters["rows_coarse"], "batches", st["batches"],
          {k: round(v[0], 1) for k, v in prof.items() if v[1] and v[0] > 0.5})
