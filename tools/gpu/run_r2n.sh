set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2n_bench.json 2>gpurun_out/r2n_bench.err; echo "bench rc=$?"
MAGNUS_BIG_PATH=direct timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2n_bench_direct.json 2>>gpurun_out/r2n_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ("r2n_bench","r2n_bench_direct"):
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["kernel_ms"])
    except Exception as e: print(f, e)
PY
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2n_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2n_gpu.log
