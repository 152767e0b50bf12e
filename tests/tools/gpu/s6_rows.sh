# Session-6: N = 4096 half-warp row passes -- parity tests first, then the same-box A/B at c5a
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knob_bitwise.py tests/test_gpu_slab.py tests/test_gpu_fullsize.py -m gpu -q -x -k "4096 or c5a or four_step or project" > gpurun_out/s6_rows_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/s6_rows_pytest.log
export EXTRA="--override batch=8" STEPS=3
bash tests/tools/gpu/ab_env.sh "c5a" "LD_PEN4_OLD=1 LD_XN_L2EF=0 LD_PEN4_ROWS_LB1=1 LD_XN_L2EF=0 LD_PEN4_ROWS_LB1=1" | tee gpurun_out/s6_ab_rows_c5a.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"pen_|flux_" --launch-count 20 --log-file gpurun_out/s6_c5a_proj_launches_rows.csv \
  env LD_HOST_NO_PIPELINE=1 python bench.py --config c5a --override batch=8 --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/s6_c5a_ncu_rows.log 2>&1; echo "ncu c5a rc=$?"
