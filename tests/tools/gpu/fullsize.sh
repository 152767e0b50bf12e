timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=5 2>&1 | grep -E "passed|failed|Error|assert|[0-9]+\.[0-9]+s call" | head -20
bash tests/tools/gpu/quick_perf.sh 2>&1 | tail -16
