# A/B of library builds in ab/*.so (LDSOLVER_LIB) on a list of configs: ms/step + kernel classes
# usage: ABLIBS="base new" CONFIGS="c2 c3" bash tests/tools/gpu/ab.sh
for rep in 1 2; do
for c in ${CONFIGS:-c2 c3}; do
for l in ${ABLIBS:-base new}; do
  LDSOLVER_LIB=$PWD/ab/lib_$l.so timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-variants ${PREC:+--precision $PREC} ${OVR:+--override $OVR} > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$rep $c %-6s'%'$l', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})
except Exception as e:
    print('$rep $c $l failed', e)
" || tail -3 gpurun_out/ab.log
done; done; done
