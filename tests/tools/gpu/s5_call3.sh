# session 5, call 3: cp.async flux_div staging, one-wave projection passes: checks + bench lines + ncu
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flux_epi.py tests/test_gpu_parity_r02.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/s5c3_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c3_pytest.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4 c3 c5b" "LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c3_ab.txt
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"flux_div|pen_" --launch-skip 10 --launch-count 4 \
  -o gpurun_out/prof_s5c3_fluxproj -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/s5c3_ncu.log 2>&1; echo "ncu rc=$?"
