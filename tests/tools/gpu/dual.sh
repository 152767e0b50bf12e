# LD_XN_DUAL A/B (two CTAs per SM hidden conv) on c2: tf32 / f16 + parity of the tf32 tests under it
for rep in 1 2; do
for d in ${DUALS:-0 1}; do
for p in ${PRECS:-tf32 f16}; do
  LD_XN_DUAL=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants --precision $p ${OVR:+--override $OVR} > gpurun_out/dual.log 2>&1
  tail -1 gpurun_out/dual.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('dual=$d $p', '%.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})
except Exception as e: print('dual=$d $p failed', e)
" || tail -3 gpurun_out/dual.log
done; done; done
LD_XN_DUAL=1 timeout 600 python -m pytest tests/test_gpu_tf32.py -x -q 2>&1 | tail -3
