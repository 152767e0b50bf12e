timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "projection or one_step" 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --precision f16 --no-cpu-baseline --no-variants > gpurun_out/bench_f16.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_f16.log').read().strip().splitlines()[-1])
print('f16', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
