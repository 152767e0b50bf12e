# Round-2 evidence in one gpurun call: GPU tests, smoke, default bench (c4), ncu launch list of the
# bench command, one `ncu --set full` capture of the hot kernels.  Everything lands in gpurun_out/.
set -u
P=${1:-tf32}
TESTS=${TESTS:-1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
if [ "$TESTS" = 1 ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 300 python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants > gpurun_out/plain_$P.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_launch_$P.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel|flux_rk|pen_" -s 40 -c 8 \
  -o gpurun_out/prof_full_$P -f python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_full_$P.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full_$P.log
