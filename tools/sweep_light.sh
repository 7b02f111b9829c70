# light rows beside the heavy path (default) vs serialised (MAGNUS_LIGHT_SIDE=0): mean and spread of the step
for i in 1 2 3; do for ls in 1 0; do
  MAGNUS_LIGHT_SIDE=$ls timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/ls_$ls.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ls_$ls.log'):
    if l.startswith('{'):
        d=json.loads(l); print('light_side=$ls', d['ms_per_step'])
"
done; done
