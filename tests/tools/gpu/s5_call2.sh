# session 5, call 2: pen_cols_r2s (coalesced column pass) check + A/B, ncu of flux_div / projection in the step's L2 state
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "projection or one_step or rollout" > gpurun_out/s5c2_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c2_pytest.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4 c3" "LD_PEN_COLS_OLD=1 LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c2_ab.txt
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"flux_div|pen_" --launch-skip 10 --launch-count 4 \
  -o gpurun_out/prof_s5_fluxproj -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/s5c2_ncu.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/s5c2_ncu.log
