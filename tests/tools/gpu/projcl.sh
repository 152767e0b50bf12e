# projection cluster-size knob (LD_PROJ_CL) x library (relaxed final cluster barrier) on c2
for l in ${ABLIBS:-dualauto projrel}; do
for cl in ${CLS:-0 2 4 8}; do
  LD_PROJ_CL=$cl LDSOLVER_LIB=$PWD/ab/lib_$l.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/pcl.log 2>&1
  tail -1 gpurun_out/pcl.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$l CL=$cl', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})
except Exception as e: print('$l $cl failed', e)
"
done; done
