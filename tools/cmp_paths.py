"""Debug: run one BASELINE config through the direct and the binned heavy path and
compare C bit for bit (both must equal the reference association)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import MagnusPlan, detect_device_params, generate  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A, B = generate.make_config_device(cfg, rp_dtype=torch.int64 if cfg == 5 else torch.int32)
sysp = detect_device_params()
res = {}
for path in ("binned", "direct"):
    os.environ["MAGNUS_HEAVY_PATH"] = path
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = MagnusPlan(A, B, sys=sysp)
        plan.ctx.profile(True)
        rp = plan.symbolic()
        C, counters = plan.numeric(rp)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        prof = plan.ctx.profile_read()
        plan.close()
        if rep == 0:
            del C
            torch.cuda.empty_cache()
        print(path, rep, f"{1e3*(t1-t0):.1f} ms", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]}, flush=True)
    # checksum of the pattern and value bits (C is too large to keep two copies)
    col = C.col.to(torch.int64)
    vb = C.val.view(torch.int64)
    w = torch.arange(col.numel(), device=col.device, dtype=torch.int64) % 1000003 + 1
    res[path] = (C.row_ptr.clone(), int((col * w).sum()), int((vb * w).sum()), int(vb.sum()))
    del C, col, vb, w
    torch.cuda.empty_cache()
a, b = res["direct"], res["binned"]
print("row_ptr equal:", bool(torch.equal(a[0], b[0])), "col checksum equal:", a[1] == b[1], "val checksum equal:",
      a[2] == b[2] and a[3] == b[3])
