# session 5, call 12: N = 4096 column pass on half-warp FFTs: parity (projection 2048 / 4096, slabs), comparison, c5a A/B
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_knob_bitwise.py -m gpu -x -q -k "projection or slab or n4096 or 2048" > gpurun_out/s5c12_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s5c12_pytest.log
for rep in 1 2; do
for e in LD_PEN4_OLD=1 LD_XN_L2EF=0; do
  env $e timeout 900 python bench.py --config c5a --override batch=8 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s5c12_c5a_$e.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/s5c12_c5a_$e.json').read().strip().splitlines()[-1]); print('c5a $e', '%.1f ms'%d['ms_per_step'], {k:(round(v['ms_per_launch']*1e3,1), round(v.get('hbm_frac',0),3)) for k,v in d['kernels'].items()})"
done; done | tee gpurun_out/s5c12_ab.txt
