# Round-2 session-6 evidence in one gpurun call: GPU tests, smoke, the default bench line, the ncu launch list of
# the bench command, one `ncu --set full` capture of the step's kernels, and one bench line per BASELINE config.
set -u
mkdir -p gpurun_out/s6_configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/s6_pytest_final.log 2>&1; echo "pytest rc=$?"
  tail -6 gpurun_out/s6_pytest_final.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke_final.log 2>&1; echo "smoke rc=$?"
  tail -3 gpurun_out/s6_smoke_final.log
fi
timeout 1200 python bench.py > gpurun_out/s6_bench_final.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s6_bench_final.log | cut -c1-400
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/s6_plain_final.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/s6_launches_final.csv env LD_HOST_NO_PIPELINE=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants \
  > gpurun_out/s6_ncu_launch_final.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_xn_kernel|flux_|pen_" --launch-skip 0 \
  --launch-count 10 -o gpurun_out/prof_s6_final -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/s6_ncu_full_final.log 2>&1; echo "ncu full rc=$?"
for c in c1 c2 c3 c4 c5b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s6_configs/$c.json 2> gpurun_out/s6_configs/$c.err
done
timeout 900 python bench.py --config c5a --override batch=8 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s6_configs/c5a.json 2> gpurun_out/s6_configs/c5a.err
echo configs done
