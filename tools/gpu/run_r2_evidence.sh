# round-2 measurement set: all GPU tests, bench lines (cfg3 with CPU baseline + e2e, the reference
# arm, cfg1/2/4), ncu launch list of cfg3 and a full capture of its top kernels
set -x
R=${R:-r2}
python -c "from paper_2501_07056_b200 import _lib; _lib.build()"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${R}_gputest.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/${R}_gputest.log
timeout 900 python bench.py > gpurun_out/${R}_bench_cfg3.json 2> gpurun_out/${R}_bench_cfg3.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_cfg3_reference_arm.json 2> gpurun_out/${R}_ref.err; echo "ref rc=$?"
for c in 1 2 4; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/${R}_bench_cfg$c.json 2>> gpurun_out/${R}_bench_small.err; echo cfg$c rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${R}_ncu.log 2>&1; echo ncu rc=$?
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_bin_big|k_bin_expand2|k_heavy_sym2|k_bin_reduce|k_rows_block|k_rows_warp" \
  --launch-skip 12 -c 7 -o gpurun_out/${R}_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/${R}_ncu_full.log 2>&1; echo ncu_full rc=$?
