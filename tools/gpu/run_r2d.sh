set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2d_parity.log 2>&1; echo "parity rc=$?"
tail -5 gpurun_out/r2d_parity.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2d_bench.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_ms"])
PY
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "cfg3_full" > gpurun_out/r2d_fullsize.log 2>&1; echo "fullsize rc=$?"
tail -3 gpurun_out/r2d_fullsize.log
