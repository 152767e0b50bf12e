# session 5, call 11: vectorised row loads in pen_rows_fwd_n256: parity + A/B + ncu
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knob_bitwise.py -m gpu -x -q -k "projection or one_step or n256" > gpurun_out/s5c11_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c11_pytest.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4" "LD_PEN_WARPFFT=1 LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c11_ab.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pen_" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/prof_s5c11_proj -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/s5c11_ncu.log 2>&1; echo "ncu rc=$?"
