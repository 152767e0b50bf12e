# Round-2 final evidence in one gpurun call: GPU tests, smoke, the default bench line, the ncu launch list of
# the bench command and one `ncu --set full` capture of the hot kernels; everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?"
  tail -6 gpurun_out/pytest_final.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"
  tail -3 gpurun_out/smoke_final.log
fi
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_final.log | cut -c1-300
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/plain_final.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_final.csv env LD_HOST_NO_PIPELINE=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel|flux_|pen_" --launch-skip 0 \
  --launch-count 11 -o gpurun_out/prof_final_r02 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
