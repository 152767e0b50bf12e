# GPU test suite (log in gpurun_out/pytest_gpu.log) + one bench line per override given as args
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head -10
bash tests/tools/gpu/variants.sh "$@"
