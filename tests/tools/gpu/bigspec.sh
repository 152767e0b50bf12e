set -x
timeout 600 python -m pytest tests/test_gpu_fno.py tests/test_gpu_tc_history.py -q -x 2>&1 | tail -2
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants"
$B > gpurun_out/r02_c4_plain.json 2>/dev/null; tail -c 400 gpurun_out/r02_c4_plain.json
$B --override fno_kmax=12,fno_layers=2,fno_width=8 > gpurun_out/r02_c4_fno.json 2>/dev/null; tail -c 300 gpurun_out/r02_c4_fno.json
$B --override tc_head=0,tc_mode=1,tc_interval=4,tc_kmax=12,tc_layers=2,tc_width=8 > gpurun_out/r02_c4_tch.json 2>/dev/null; tail -c 300 gpurun_out/r02_c4_tch.json
