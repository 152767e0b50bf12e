# session 5, call 10: N = 256 half-warp FFT projection passes: parity, knob tests, A/B vs the warp-FFT passes, ncu
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "projection or one_step or rollout" > gpurun_out/s5c10_pytest.log 2>&1; echo "pytest parity rc=$?"
tail -3 gpurun_out/s5c10_pytest.log
timeout 1200 python -m pytest tests/test_gpu_knob_bitwise.py tests/test_gpu_parity_r02.py -m gpu -x -q -k "n256 or 256 or c4 or shard" > gpurun_out/s5c10_pytest2.log 2>&1; echo "pytest knob rc=$?"
tail -3 gpurun_out/s5c10_pytest2.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4" "LD_PEN_WARPFFT=1 LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c10_ab.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pen_" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/prof_s5c10_proj -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/s5c10_ncu.log 2>&1; echo "ncu rc=$?"
# first-layer gather order on the same box at c5b / c4 (the per-config runs of two boxes disagreed)
for rep in 1 2; do
for e in LD_XN_GATHER_Y=1 LD_XN_L2EF=0; do
  env $e timeout 600 python bench.py --config c5b --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s5c10_c5b_$e.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/s5c10_c5b_$e.json').read().strip().splitlines()[-1]); print('c5b $e', '%.3f ms'%d['ms_per_step'], {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})"
done; done | tee gpurun_out/s5c10_gather.txt
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4" "LD_XN_GATHER_Y=1 LD_XN_L2EF=0" 2>&1 | tee -a gpurun_out/s5c10_gather.txt
