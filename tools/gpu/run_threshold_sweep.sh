# fine chunk width and sort-vs-dense reducer threshold on B200, times + ncu counters
set -x
M="gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum"
: > gpurun_out/thr_sweep.jsonl
timeout 900 python tools/threshold_sweep.py --lines 4,32,128,256,1024 --tag chunk_width >> gpurun_out/thr_sweep.jsonl 2> gpurun_out/thr_sweep.err; echo "width rc=$?"
for v in binE128 binE256 base; do
  PHASE_LIB=$PWD/variants/lib_$v.so timeout 600 python tools/threshold_sweep.py --lines 128 --tag kBinE_$v >> gpurun_out/thr_sweep.jsonl 2>> gpurun_out/thr_sweep.err; echo "$v rc=$?"
done
for line in 32 128 256; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/thr_ncu_line$line.csv \
    python tools/threshold_sweep.py --lines $line --reps 1 --warmup 0 > /dev/null 2>> gpurun_out/thr_sweep.err; echo "ncu line $line rc=$?"
done
for v in binE128 binE256; do
  PHASE_LIB=$PWD/variants/lib_$v.so timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/thr_ncu_$v.csv \
    python tools/threshold_sweep.py --lines 128 --reps 1 --warmup 0 > /dev/null 2>> gpurun_out/thr_sweep.err; echo "ncu $v rc=$?"
done
cat gpurun_out/thr_sweep.jsonl
