# A/B of variants/lib_*.so on cfg3 (bench.py, no CPU / e2e legs); alternating order exposes noise
cp paper_2501_07056_b200/libmagnus_b200.so /tmp/lib_orig.so
for v in ${VARIANTS:-base s6b0 s6b16 s8b16 s5b8 base s6b16}; do
  cp variants/lib_$v.so paper_2501_07056_b200/libmagnus_b200.so
  timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/var_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/var_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernel_ms']; print('$v', d['ms_per_step'], round(sum(k.values()),1), 'sym_heavy', k['sym_heavy'], 'expand', k['bin_expand'], 'big', k['bin_big'], 'red', k['bin_reduce'])
" || tail -3 gpurun_out/var_$v.log
done
cp /tmp/lib_orig.so paper_2501_07056_b200/libmagnus_b200.so
