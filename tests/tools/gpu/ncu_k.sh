# ncu --set full of selected kernels of one bench run: ncu_k.sh <config> <regex> <skip> <count> <tag>
C=${1:-c4}; K=${2:-flux_rk}; S=${3:-0}; N=${4:-2}; T=${5:-k}
mkdir -p gpurun_out
timeout 300 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/plain_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip $S --launch-count $N \
  -o gpurun_out/prof_$T -f python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-variants \
  > gpurun_out/ncu_$T.log 2>&1; echo "ncu $T rc=$?"
