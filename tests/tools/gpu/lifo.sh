# LIFO tile order (default) vs forward order (LD_LIFO=0) per config
for rep in 1 2; do
for c in ${CONFIGS:-c3 c4}; do
for lf in 1 0; do
  LD_LIFO=$lf timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/lifo.log 2>&1
  tail -1 gpurun_out/lifo.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$c lifo=$lf', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items() if v['ms_per_launch']})
except Exception as e: print('$c $lf failed', e)
"
done; done; done
