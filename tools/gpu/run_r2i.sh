set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 600 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/r2i_bench4.json 2>gpurun_out/r2i.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2i_bench4.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_ms"])
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rows_warp" -c 2 -o gpurun_out/r2i_warp python bench.py --config 4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2i_ncu.log 2>&1; echo ncu rc=$?
timeout 600 nsys --version 2>/dev/null; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo launches rc=$?
