# session 5, call 7: first-layer x-fastest gather and the contiguous-tile output layer (flux epilogue): checks + A/B
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_knob_bitwise.py -m gpu -x -q -k "GATHER" > gpurun_out/s5c7_pytest.log 2>&1; echo "pytest gather rc=$?"
tail -2 gpurun_out/s5c7_pytest.log
LD_XN_CT_OUT=1 timeout 900 python -m pytest tests/test_gpu_flux_epi.py tests/test_gpu_parity_r02.py -m gpu -x -q -k "not c5b" > gpurun_out/s5c7_pytest_ct.log 2>&1; echo "pytest ct_out rc=$?"
tail -2 gpurun_out/s5c7_pytest_ct.log
for rep in 1 2; do
STEPS=10 bash tests/tools/gpu/ab_env.sh "c4 c3" "LD_XN_GATHER_Y=1 LD_XN_CT_OUT=1 LD_XN_L2EF=0" 2>&1
done | tee gpurun_out/s5c7_ab.txt
