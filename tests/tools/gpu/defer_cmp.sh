timeout 200 python tests/tools/tc_quick.py 2>&1 | tail -9
for d in 0 64; do for p in tf32 f16; do
LD_TC_DEBUG=$d timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline > gpurun_out/bd_$p_$d.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bd_$p_$d.log').read().strip().splitlines()[-1])
print('dbg=$d', '$p', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
done; done
