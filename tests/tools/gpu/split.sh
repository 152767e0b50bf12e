# batch split over two streams (LD_SPLIT=2) vs one stream (LD_SPLIT=0) on c2
for rep in 1 2; do
for sp in 0 2; do
  LD_SPLIT=$sp timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants ${EXTRA} > gpurun_out/split.log 2>&1
  tail -1 gpurun_out/split.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('split=$sp', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items() if v['ms_per_launch']})
except Exception as e: print('split=$sp failed', e)
" || tail -3 gpurun_out/split.log
done; done
