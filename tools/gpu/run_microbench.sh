# building-block microbenchmarks (reference bench.py:88-196) over chunk counts; best of 3
for c in 64 256 1024 4096; do python -m paper_2501_07056_b200.cli microbench --size 67108864 --length 1048576 --chunks $c --reps 3 --json 2>/dev/null; done > gpurun_out/r2_microbench.jsonl
python - <<'PY'
import json, collections
best = collections.defaultdict(dict)
for l in open("gpurun_out/r2_microbench.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l); c = d["params"]["n_chunks"]; b = d["benchmark"]
    best[c][b] = min(best[c].get(b, 1e9), d["seconds"])
print("chunks   histogram  prefix_sum     reorder dense_accum  sort_accum      stream       total   total/stream")
for c in sorted(best):
    r = best[c]
    print(f"{c:6d} " + " ".join(f"{1e3*r[k]:9.3f}ms" for k in ("histogram","prefix_sum","reorder","dense_accum","sort_accum","stream","total")) + f"   {r['total']/r['stream']:8.1f}x")
PY
