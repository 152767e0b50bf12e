# conv_tc time under the LD_TC_DEBUG knobs (measurement only): 0 full, 1 no loads, 2 no epilogue, 4 no MMA, 3, 6, 5, 7
for d in 0 1 2 4 3 6 5 7; do
  LD_TC_DEBUG=$d timeout 120 python bench.py --steps 10 --warmup 3 --precision f16 --no-cpu-baseline > gpurun_out/knob_$d.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/knob_$d.log').read().strip().splitlines()[-1])
print('dbg=$d', {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})" 2>/dev/null || (echo "dbg=$d failed"; tail -3 gpurun_out/knob_$d.log)
done
