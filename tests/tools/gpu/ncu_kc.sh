# ncu --set full of kernels matching $1 (regex) in the bench of config $2, skip $3, count $4
K=$1; CFG=${2:-c2}; S=${3:-20}; C=${4:-2}
timeout 300 python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/plain_kc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $C \
  -o gpurun_out/prof_kc python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu_kc.log 2>&1; echo "ncu rc=$?"
