"""Per-product cost of the heavy-path kernels against the size of B (R-MAT 2^17..2^20, ef 16): does the
L2 residency of B (126 MB of L2) matter?  Prints ps per heavy product per kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import MagnusPlan, _lib, detect_device_params, generate  # noqa: E402

for scale in (17, 18, 19, 20):
    A = generate.rmat_device(scale, 16, seed=3)
    sysp = detect_device_params()
    for r in range(3):
        plan = MagnusPlan(A, A, sys=sysp)
        plan.ctx.profile(True)
        rp = plan.symbolic()
        C, cnt = plan.numeric(rp)
        torch.cuda.synchronize()
        prof = plan.ctx.profile_read()
        hs = plan.ctx.heavy_stats()
        plan.close()
        del C, rp
        torch.cuda.empty_cache()
    tot = hs["big_products"] + hs["small_products"]
    print(f"2^{scale}: B {A.col.numel() * 12 / 1e6:.0f} MB, {tot:.3e} heavy products;",
          {k: round(1e9 * v[0] / tot, 2) for k, v in prof.items() if k in ("sym_heavy", "bin_expand", "bin_big", "bin_reduce")},
          "ps per heavy product", flush=True)
    del A
    _lib.release_workspace()
    torch.cuda.empty_cache()
