for w in 5 0 5 0; do
  BENCH_SAMPLER_WAIT=$w timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/smp_$w.log 2>&1
  python -c "
import json
for l in open('gpurun_out/smp_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); print('wait=$w', d['ms_per_step'], d['clocks'])
"
done
