# quick check of the conv/flux path: TF32/F16 parity tests, then a short bench
timeout 600 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xn.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_xn.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.4g ms/step %.4f e2e %.4g'%(d['value'],d['ms_per_step'],d['e2e']['value']))
print({k:(round(v['ms_per_launch']*1e3,2),round(v['share_of_step'],3)) for k,v in d['kernels'].items()})
print('roofline',d['roofline']['kernel'],round(d['roofline']['achieved'],1),round(d['roofline']['frac'],3))
print('variants',{k:(round(v['ms_per_step'],4)) for k,v in d['variants'].items()})
" || tail -30 gpurun_out/bench_xn.log
if [ "${NCU:-0}" = "1" ]; then
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/plain_xn.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel|flux_rk|proj_fused|conv_first" -s 60 -c 8 \
  -o gpurun_out/prof_xn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu_xn.log 2>&1; echo "ncu rc=$?"
fi
