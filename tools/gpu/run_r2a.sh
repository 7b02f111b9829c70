set -x
nproc; free -g | head -2
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 2400 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_gpu_tests.log
timeout 3000 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r2_fullsize.log 2>&1; echo "fullsize rc=$?"
tail -30 gpurun_out/r2_fullsize.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench.json
