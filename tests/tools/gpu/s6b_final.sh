# Round-2 session-6 evidence in one gpurun call: GPU tests, smoke, the default bench line, the ncu launch list of
set -u
mkdir -p gpurun_out/s6b_configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/s6b_pytest_final.log 2>&1; echo "pytest rc=$?"
  tail -6 gpurun_out/s6b_pytest_final.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6b_smoke_final.log 2>&1; echo "smoke rc=$?"
  tail -3 gpurun_out/s6b_smoke_final.log
fi
timeout 1200 python bench.py > gpurun_out/s6b_bench_final.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s6b_bench_final.log | cut -c1-400
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/s6b_plain_final.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/s6b_launches_final.csv env LD_HOST_NO_PIPELINE=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants \
  > gpurun_out/s6b_ncu_launch_final.log 2>&1; echo "ncu launches rc=$?"
for c in c1 c2 c3 c4 c5b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s6b_configs/$c.json 2> gpurun_out/s6b_configs/$c.err
done
timeout 900 python bench.py --config c5a --override batch=8 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s6b_configs/c5a.json 2> gpurun_out/s6b_configs/c5a.err
echo configs done
