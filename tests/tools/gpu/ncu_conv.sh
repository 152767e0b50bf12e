# ncu --set full of one hidden conv launch (and the last layer) at a config: ncu_conv.sh c4 tf32
C=${1:-c4}; P=${2:-tf32}
mkdir -p gpurun_out
timeout 300 python bench.py --config $C --precision $P --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/plain_conv_$C.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_xn_kernel --launch-skip 1 --launch-count 5 \
  -o gpurun_out/prof_conv_${C}_$P -f python bench.py --config $C --precision $P --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_conv_${C}_$P.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_conv_${C}_$P.log
