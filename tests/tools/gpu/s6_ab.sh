# Session-6 A/B on one box: the N = 4096 half-warp column pass (default) vs LD_PEN4_OLD=1 (64 x 64 shuffle-FFT form)
# at c5a (batch 8 on one GPU), twice each, plus an ncu launch list of one c5a step's projection passes.
set -u
mkdir -p gpurun_out
export EXTRA="--override batch=8" STEPS=3
bash tests/tools/gpu/ab_env.sh "c5a" "LD_PEN4_OLD=1 LD_XN_L2EF=0 LD_PEN4_OLD=1 LD_XN_L2EF=0" | tee gpurun_out/s6_ab_c5a.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"pen_|flux_" --launch-count 20 --log-file gpurun_out/s6_c5a_proj_launches.csv \
  env LD_HOST_NO_PIPELINE=1 python bench.py --config c5a --override batch=8 --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/s6_c5a_ncu.log 2>&1; echo "ncu c5a rc=$?"
