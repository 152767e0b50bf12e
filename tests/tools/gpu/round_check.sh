# Round evidence in one gpurun call: GPU tests, smoke, headline bench, ncu launch list,
# one `ncu --set full` capture of the hot kernels.  Everything lands in gpurun_out/.
set -u
P=${1:-tf32}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke.log | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log | cut -c1-600
timeout 300 python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants > gpurun_out/plain_$P.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_launch_$P.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel|flux_rk|proj|conv_first" -s 40 -c 6 \
  -o gpurun_out/prof_full_$P python bench.py --steps 2 --warmup 3 --precision $P --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_full_$P.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full_$P.log
