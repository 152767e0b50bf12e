# one ncu --set full capture of the kernels matching $2 (regex), after a plain run of the same command
P=${1:-f16}; K=${2:-conv_tc_kernel}; S=${3:-6}; C=${4:-1}
python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline > gpurun_out/plainf_$P.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/prof_${K}_$P python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline > gpurun_out/ncuf_$P.log 2>&1
tail -3 gpurun_out/ncuf_$P.log
