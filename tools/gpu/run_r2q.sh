set -x
MAGNUS_BIG_PATH=direct timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_bd_num" -c 1 -o gpurun_out/r2q_bd python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2q_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/r2q_ncu.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_bin_big" -c 1 --launch-skip 2 -o gpurun_out/r2q_big python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2q_ncu2.log 2>&1; echo ncu rc=$?
