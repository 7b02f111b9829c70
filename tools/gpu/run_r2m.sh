set -x
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_heavy_sym2" -c 1 -o gpurun_out/r2m_sym2 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2m_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/r2m_ncu.log
