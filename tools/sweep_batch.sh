# reorder-buffer batch fraction sweep on cfg3 (MAGNUS_BATCH_FRAC), alternating to expose run-to-run noise
for f in ${FRACS:-0.3 0.2 0.3 0.2 0.25}; do
  MAGNUS_BATCH_FRAC=$f timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/sw_$f.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/sw_$f.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print('$f', d['ms_per_step'], round(sum(k.values()),1), k['bin_expand'], k['bin_big'], k['bin_reduce'], k['num_warp'])
" || tail -3 gpurun_out/sw_$f.log
done
