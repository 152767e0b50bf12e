# Session 6: the packed-fp32 first layer (default) vs the tcgen05 first layer (LD_FIRST_TC=1), its tests, and
# the fair TMA fill microbenchmark (tests/tools/tma_fair_microbench.cu).
set -u
mkdir -p gpurun_out/s6
for k in 0 1; do
  if [ $k = 1 ]; then export LD_PEN4_OLD=1; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -k "projection_parity and 4096" -q -rfs > gpurun_out/s6/pen4_old$k.log 2>&1; echo "pen4 old=$k rc=$?"
  tail -2 gpurun_out/s6/pen4_old$k.log
done
unset LD_PEN4_OLD
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/s6/tma_fair tests/tools/tma_fair_microbench.cu -lcuda && \
  timeout 120 gpurun_out/s6/tma_fair > gpurun_out/s6/tma_fair.log 2>&1; echo "tma rc=$?"; cat gpurun_out/s6/tma_fair.log
timeout 1500 python -m pytest tests/test_gpu_knob_bitwise.py -k "first_layer or GATHER" tests/test_gpu_tf32.py tests/test_gpu_parity_r02.py tests/test_gpu_flux_epi.py -q -rfs -x > gpurun_out/s6/pytest_first.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/s6/pytest_first.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-variants --no-cpu-baseline > gpurun_out/s6/bench_f2_$i.json 2> gpurun_out/s6/bench_f2_$i.err
  timeout 600 env LD_FIRST_TC=1 python bench.py --steps 20 --warmup 5 --no-variants --no-cpu-baseline > gpurun_out/s6/bench_tc_$i.json 2> gpurun_out/s6/bench_tc_$i.err
done
python - <<'PY'
import json
for t in ("f2_1", "tc_1", "f2_2", "tc_2"):
    try:
        d = json.loads(open(f"gpurun_out/s6/bench_{t}.json").read().strip().splitlines()[-1])
        k = d["kernels"]
        print(t, "ms/step %.3f" % d["ms_per_step"], "first %.1f us" % (k["conv_first"]["ms_per_launch"] * 1e3),
              "hidden %.1f us" % (k["conv_hidden"]["ms_per_launch"] * 1e3), "clk", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(t, "ERR", e)
PY
