timeout 900 python -m pytest tests/test_gpu_gustavson.py tests/test_gpu_microbench.py tests/test_cli.py -x -q -m gpu 2>&1 | tail -3
python - <<'PY'
import os, time, torch
from paper_2501_07056_b200 import generate, gustavson_esc
A = generate.rmat_device(17, 16, seed=3)
for mode in ("device", "cub", "device", "cub"):
    if mode == "cub": os.environ["MAGNUS_ESC_SORT"] = "cub"
    else: os.environ.pop("MAGNUS_ESC_SORT", None)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = gustavson_esc(A, A)
    torch.cuda.synchronize(); print("esc", mode, round(1e3 * (time.perf_counter() - t0), 1), "ms", r.counters)
PY
