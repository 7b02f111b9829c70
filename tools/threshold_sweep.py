"""Re-derivation of the two execution parameters of the fine level on B200:

* the fine chunk width (n_chunks_fine of the numeric plan, planner.py:106-152), swept through
  SystemParams.cache_line_bytes (the only parameter the chunk count depends on once the span fits);
* the device's sort-vs-dense reducer threshold kBinE (chunks with at most kBinE products go to the
  sort-style reducer, the others to the dense accumulator), swept through variant builds
  (tools/build_variants.sh ... "-DMG_BIN_E=...", selected with PHASE_LIB).

One product of a BASELINE config per setting; prints one JSON line per setting with the step time,
the per-kernel event times and the heavy-row chunk statistics.  Run it under
`ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum`
with --reps 1 --warmup 0 for the counters behind the times (tools/gpu/run_threshold_sweep.sh).
Values differ between chunk widths only by the association the reference itself would use with those
parameters; every setting is checked for a clean status, not against the oracle (tests do that)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import _lib  # noqa: E402

if os.environ.get("PHASE_LIB"):
    _lib.LIB_PATH = os.environ["PHASE_LIB"]
from paper_2501_07056_b200 import MagnusPlan, SystemParams, compute_chunk_plan, generate  # noqa: E402
from paper_2501_07056_b200.planner import NUMERIC  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--lines", default="128")          # cache_line_bytes values, comma separated
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--tag", default="")
args = ap.parse_args()

A, B = generate.make_config_device(args.config, rp_dtype=torch.int64 if args.config == 5 else torch.int32)
for line in (int(x) for x in args.lines.split(",")):
    sysp = SystemParams(cache_line_bytes=line, l2_bytes=232448, memory_budget_bytes=40 << 30)
    plan_n = compute_chunk_plan(sysp, B.n_cols, NUMERIC)
    best, prof_best, stats = None, None, None
    for r in range(args.warmup + args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = MagnusPlan(A, B, sys=sysp)
        plan.ctx.profile(True)
        rp = plan.symbolic()
        C, counters = plan.numeric(rp)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        prof = plan.ctx.profile_read()
        if stats is None:
            stats = plan.ctx.heavy_stats()
        plan.close()
        del C
        if r >= args.warmup and (best is None or t1 - t0 < best):
            best, prof_best = t1 - t0, prof
    print(json.dumps({"tag": args.tag, "config": args.config, "cache_line_bytes": line,
                      "n_chunks_fine": plan_n.n_chunks_fine, "chunk_len_fine": plan_n.chunk_len_fine,
                      "ms_per_product": round(1e3 * best, 2),
                      "kernel_ms": {k: round(v[0], 2) for k, v in prof_best.items() if v[1]},
                      "heavy_chunks": stats, "nnz_c": counters["nnz_c"]}), flush=True)
