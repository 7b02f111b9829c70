set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2j_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2j_gpu.log
for c in 3 4; do
timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2j_bench$c.json 2>>gpurun_out/r2j_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/r2j_bench$c.json").read().strip().splitlines()[-1]); print($c, d["ms_per_step"], d["kernel_ms"])
PY
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "cfg4 or cfg3_full" > gpurun_out/r2j_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/r2j_full.log
