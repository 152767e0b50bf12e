for cl in 0 8 0 8; do
  LD_FUSED_CL=$cl LDSOLVER_LIB=$PWD/ab/lib_fusedcl.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/fcl.log 2>&1
  tail -1 gpurun_out/fcl.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('CL=$cl', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
done
