set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-against_oracle or hot_chunks or heavy_paths or heavy_rows_1024 or reference_golden}" > gpurun_out/ab_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/ab_gpu.log
bash tools/sweep_variants.sh
