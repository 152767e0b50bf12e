# round profile: bench (headline tf32 + variants), launch list, one full capture of each kernel class
P=${1:-tf32}
python bench.py --steps 20 --warmup 5 --precision $P > gpurun_out/bench_round_$P.log 2>&1
tail -1 gpurun_out/bench_round_$P.log | cut -c1-400
python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline --no-variants > gpurun_out/plain_$P.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline --no-variants > gpurun_out/ncu_launch_$P.log 2>&1
python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline --no-variants > gpurun_out/plain2_$P.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"conv_tc_kernel|flux_rk|proj_fused|conv_first" -s 22 -c 5 -o gpurun_out/prof_round_$P python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline --no-variants > gpurun_out/ncu_full_$P.log 2>&1
tail -2 gpurun_out/ncu_full_$P.log
