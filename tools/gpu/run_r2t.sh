set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "against_oracle or hot_chunks or heavy_paths or heavy_rows_1024" > gpurun_out/r2t_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2t_gpu.log
VARIANTS="inv1 inv0 inv1 inv0" bash tools/sweep_variants.sh
