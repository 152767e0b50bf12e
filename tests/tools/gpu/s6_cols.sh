# Session-6: N = 4096 column pass with two CTAs per SM (default) vs LD_PEN4_COLS_LB1=1 -- parity tests, then the A/B at c5a
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knob_bitwise.py tests/test_gpu_slab.py tests/test_gpu_fullsize.py -m gpu -q -x -k "4096 or c5a or four_step or project" > gpurun_out/s6_cols_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/s6_cols_pytest.log
export EXTRA="--override batch=8" STEPS=3
bash tests/tools/gpu/ab_env.sh "c5a" "LD_PEN4_COLS_LB1=1 LD_XN_L2EF=0 LD_PEN4_COLS_LB1=1 LD_XN_L2EF=0" | tee gpurun_out/s6_ab_cols_c5a.txt
