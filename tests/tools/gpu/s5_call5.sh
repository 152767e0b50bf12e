# session 5, call 5: sequential-chunk host pipeline (e2e) A/B + bitwise test; c5a projection per-pass launch list
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_r02.py tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/s5c5_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c5_pytest.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4 c3" "LD_HOST_CONCURRENT=1 LD_XN_L2EF=0" 2>&1
done > gpurun_out/s5c5_ab.txt
for f in gpurun_out/ab_c4_LD_HOST_CONCURRENT_1.json gpurun_out/ab_c4_LD_XN_L2EF_0.json gpurun_out/ab_c3_LD_HOST_CONCURRENT_1.json gpurun_out/ab_c3_LD_XN_L2EF_0.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', 'value %.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
done | tee -a gpurun_out/s5c5_ab.txt
cat gpurun_out/s5c5_ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"pen_" \
  --log-file gpurun_out/launches_c5a.csv env LD_HOST_NO_PIPELINE=1 python bench.py --config c5a --override batch=8 --steps 1 --warmup 1 --no-variants --no-cpu-baseline \
  > gpurun_out/s5c5_ncu.log 2>&1; echo "ncu rc=$?"
