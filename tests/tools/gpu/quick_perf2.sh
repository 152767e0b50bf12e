timeout 200 python tests/tools/tc_quick.py > gpurun_out/tc_quick.log 2>&1; tail -9 gpurun_out/tc_quick.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tf32.py -x -q 2>&1 | tail -2
bash tests/tools/gpu/quick_perf.sh 2>&1 | tail -16
