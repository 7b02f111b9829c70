set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2f_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/r2f_parity.log
VARIANTS="g4m4 g2m5 g2m4 g4m4u2 g4m4" bash tools/sweep_variants.sh
