set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "device_coarse_level or against_oracle or reference_golden" > gpurun_out/r2r_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -30 gpurun_out/r2r_gpu.log
