set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1800 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2b_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r2b_gpu_tests.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "cfg3_full or cfg5" > gpurun_out/r2b_fullsize.log 2>&1; echo "fullsize rc=$?"
tail -15 gpurun_out/r2b_fullsize.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
