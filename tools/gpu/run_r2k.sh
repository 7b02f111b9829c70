set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 600 python -m pytest tests/test_waves.py -x -q > gpurun_out/r2k_waves.log 2>&1; echo "waves rc=$?"
tail -3 gpurun_out/r2k_waves.log
timeout 1200 python bench.py --config 5 --steps 1 --warmup 0 > gpurun_out/r2k_bench5.json 2> gpurun_out/r2k_bench5.err; echo "bench5 rc=$?"
tail -c 1500 gpurun_out/r2k_bench5.json; tail -5 gpurun_out/r2k_bench5.err
