"""Ablation on B200: MAGNUS (locality generation) vs the Gustavson baselines
(full-width dense accumulator, expand-sort-compress) on the BASELINE configs.
Device-resident inputs, one warm-up call, wall time around each synchronised call (best of reps),
GFLOP/s = 2 x products / t.  Prints one JSON line per (config, algorithm)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2501_07056_b200 import generate, gustavson_dense, gustavson_esc, spgemm_magnus  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "4", "3"])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
algos = sys.argv[3].split(",") if len(sys.argv) > 3 else ["magnus", "dense", "esc"]
FN = {"magnus": spgemm_magnus, "dense": gustavson_dense, "esc": gustavson_esc}
for cfg in cfgs:
    A, B = generate.make_config_device(cfg)
    first = None
    for algo in algos:
        best = None
        FN[algo](A, B)   # warm-up: workspace pools and the C allocation are cached afterwards
        torch.cuda.synchronize()
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = FN[algo](A, B)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            prods, nnz = res.counters["inter_prod_size"], res.counters["nnz_c"]
            if first is None:
                first = (res.C.row_ptr[-1].item(), res.C.col[:: max(1, nnz // 4096)].clone())
            else:
                assert res.C.row_ptr[-1].item() == first[0] and torch.equal(res.C.col[:: max(1, nnz // 4096)], first[1])
            del res
        torch.cuda.empty_cache()
        print(json.dumps({"config": cfg, "algo": algo, "s": round(best, 4), "gflops": round(2 * prods / best / 1e9, 2),
                          "products": prods, "nnz_c": nnz}), flush=True)
    del A, B
    torch.cuda.empty_cache()
