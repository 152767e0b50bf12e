# source-level warp sampling of one hidden conv launch at a larger batch (more samples)
O=${1:-batch=128}; [ "$O" = "none" ] && O=""
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants ${O:+--override $O} > gpurun_out/plain_s.log 2>&1 && \
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on \
  -k regex:conv_xn_kernel -s 56 -c 1 -o gpurun_out/prof_src python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants ${O:+--override $O} > gpurun_out/ncu_s.log 2>&1; echo "ncu rc=$?"
