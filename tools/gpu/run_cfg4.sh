for i in 1 2 3; do
timeout 300 python bench.py --config 4 --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cfg4', d['ms_per_step'], d['kernel_ms'])
"
done
MAGNUS_TRACE=1 python tools/phase_time.py 4 3 2>&1 | tail -24
