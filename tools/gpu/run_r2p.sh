set -x
MAGNUS_BIG_PATH=fused timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_fu_sweep" -c 1 -o gpurun_out/r2p_fu python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2p_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/r2p_ncu.log
