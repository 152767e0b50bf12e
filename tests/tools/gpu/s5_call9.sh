# session 5, call 9: output layer (flux epilogue) with 8 positions per tile: bitwise vs the 4-position strip form, parity, A/B
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_knob_bitwise.py -m gpu -x -q -k "CT_OUT" > gpurun_out/s5c9_pytest_bw.log 2>&1; echo "pytest bitwise rc=$?"
tail -2 gpurun_out/s5c9_pytest_bw.log
timeout 1500 python -m pytest tests/test_gpu_flux_epi.py tests/test_gpu_parity_r02.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/s5c9_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c9_pytest.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4 c3" "LD_XN_NO_CT_OUT=1 LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c9_ab.txt
