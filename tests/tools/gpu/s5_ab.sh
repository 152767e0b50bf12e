# Round-2 session-5 quick check + A/B: projection / slab / flux-epilogue GPU tests, then c4 / c3 bench lines
# for the fused inverse+correction projection pass and the L2 evict_first knob
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r02.py tests/test_gpu_slab.py tests/test_gpu_flux_epi.py -m gpu -x -q > gpurun_out/s5_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s5_pytest.log
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4" "LD_PROJ_UNFUSED=1 LD_XN_L2EF=0 LD_XN_L2EF=1 LD_XN_L2EF=2 LD_XN_L2EF=3" 2>&1 | tee gpurun_out/s5_ab_c4.txt
STEPS=10 bash tests/tools/gpu/ab_env.sh "c3 c5b" "LD_PROJ_UNFUSED=1 LD_XN_L2EF=0 LD_XN_L2EF=1" 2>&1 | tee gpurun_out/s5_ab_c3c5b.txt
