# clock sampler period A/B: does nvidia-smi polling perturb the timed step?
for ms in 100 500 100 500 1000 100; do
  BENCH_SAMPLER_MS=$ms timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/smp_$ms.log 2>&1
  python -c "
import json
for l in open('gpurun_out/smp_$ms.log'):
    if l.startswith('{'):
        d=json.loads(l); print('period_ms=$ms', d['ms_per_step'], d['clocks']['samples'])
"
done
