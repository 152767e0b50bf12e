# ncu --set full of kernels matching $1 (regex), skip $2, count $3; tf32 bench, no variants
K=$1; S=${2:-20}; C=${3:-2}
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $C \
  -o gpurun_out/prof_k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"
