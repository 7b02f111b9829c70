set -x
MAGNUS_BIG_W2=3 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "against_oracle or hot_chunks or heavy_paths or heavy_rows_1024 or reference_golden" > gpurun_out/w2_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/w2_gpu.log
for w in 0 3 2 1 0 3; do
MAGNUS_BIG_W2=$w timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/w2_$w.log 2>&1
python -c "
import json
for l in open('gpurun_out/w2_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print('w2=$w', d['ms_per_step'], 'expand', k['bin_expand'], 'big', k['bin_big'], 'red', k['bin_reduce'])
" || tail -3 gpurun_out/w2_$w.log
done
