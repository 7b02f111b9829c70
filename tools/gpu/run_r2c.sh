set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
MAGNUS_BD_ORDER=arrival timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2c_bench_arrival.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/r2c_bench_arrival.json"]:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["kernel_ms"])
PY
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_bd_num" -c 2 -o gpurun_out/r2c_bd python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2c_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/r2c_ncu.log
