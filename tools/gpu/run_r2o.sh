set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "direct_big_chunk and fused" > gpurun_out/r2o_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r2o_gpu.log
MAGNUS_BIG_PATH=fused timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2o_bench_fused.json 2>gpurun_out/r2o_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/r2o_bench.err
python - <<'PY'
import json
for f in ("r2o_bench_fused",):
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["kernel_ms"])
    except Exception as e: print(f, e)
PY
