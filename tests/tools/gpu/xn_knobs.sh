# conv_xn per-launch time under the LD_XN_DEBUG knobs (measurement build, -DLD_XN_KNOBS):
# 0 full, 1 no A copies, 2 no epilogue, 4 no MMA, 8 no W copies, and combinations
P=${1:-tf32}
LD_NVCC_EXTRA=-DLD_XN_KNOBS python -c "from paper_2507_01975_b200 import build as B; B.build(force=True)" || exit 1
for d in ${KNOBS:-0 1 8 9 2 4 6 3 5 12 13}; do
  LD_XN_DEBUG=$d timeout 120 python bench.py --steps 10 --warmup 3 --precision $P --no-cpu-baseline --no-variants > gpurun_out/xnknob_$d.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/xnknob_$d.log').read().strip().splitlines()[-1])
print('dbg=$d', {k:round(v['ms_per_launch']*1e3,1) for k,v in d['kernels'].items()})" 2>/dev/null || (echo "dbg=$d failed"; tail -3 gpurun_out/xnknob_$d.log)
done
