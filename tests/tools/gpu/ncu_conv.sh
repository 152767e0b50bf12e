# one ncu --set full capture of a hidden tcgen05 conv launch (after a plain run of the same command)
P=${1:-tf32}
timeout 300 python bench.py --steps 1 --warmup 3 --precision $P --no-cpu-baseline --no-variants > gpurun_out/plain_conv.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_xn_kernel -s 56 -c 1 \
  -o gpurun_out/prof_conv_$P python bench.py --steps 1 --warmup 3 --precision $P --no-cpu-baseline --no-variants > gpurun_out/ncu_conv.log 2>&1; echo "ncu rc=$?"
