# session 5, call 8: chunk stream priorities in the host pipeline (e2e) A/B; knob bitwise tests; conv_first ncu
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_knob_bitwise.py tests/test_gpu_parity_r02.py -m gpu -x -q -k "host or CT_OUT or bitwise or shard" > gpurun_out/s5c8_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c8_pytest.log
for rep in 1 2; do
for c in c4 c3 c5b; do for e in LD_HOST_NO_PRIO=1 LD_XN_L2EF=0; do
  env $e timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s5c8_${c}_$e.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/s5c8_${c}_$e.json').read().strip().splitlines()[-1]); print('$c $e', 'value %.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ratio %.3f'%(d['e2e']['value']/d['value']))"
done; done; done | tee gpurun_out/s5c8_ab.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel" --launch-skip 0 --launch-count 1 \
  -o gpurun_out/prof_s5c8_first -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/s5c8_ncu.log 2>&1; echo "ncu rc=$?"
