# full GPU test suite, then quick_perf
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
bash tests/tools/gpu/quick_perf.sh
