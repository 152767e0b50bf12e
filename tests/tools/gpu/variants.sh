# bench kernel times for a list of measurement overrides (one bench line each)
for o in "${@}"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants ${PREC:+--precision $PREC} ${o:+--override $o} > gpurun_out/var.log 2>&1
  tail -1 gpurun_out/var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%-28s'%'$o', 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/var.log
done
