# round-end measurement set: bench lines of cfg1-4 (cfg3 with CPU baseline and e2e), ncu launch list of cfg3
for c in 3 1 2 4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_cfg$c.log 2>&1; echo cfg$c rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_bin_big|k_bin_expand2|k_heavy_sym2|k_bin_reduce" \
  --launch-skip 9 -c 5 -o gpurun_out/full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
