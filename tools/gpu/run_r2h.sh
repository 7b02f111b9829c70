set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2h_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2h_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2h_bench.json 2>gpurun_out/r2h_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2h_bench.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_ms"])
PY
MAGNUS_BIG_PATH=direct timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2h_bench_direct.json 2>>gpurun_out/r2h_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2h_bench_direct.json").read().strip().splitlines()[-1]); print("direct", d["ms_per_step"], d["kernel_ms"])
PY
