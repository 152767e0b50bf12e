# conv_xn per-phase timestamps (measurement build) for a few knob settings
LD_NVCC_EXTRA=-DLD_XN_KNOBS python -c "from paper_2507_01975_b200 import build as B; B.build(force=True)" || exit 1
for d in ${KNOBS:-64 125}; do
  echo "== LD_XN_DEBUG=$d"
  LD_XN_DEBUG=$d LD_NO_GRAPH=1 timeout 120 python bench.py --steps 1 --warmup 1 --precision ${P:-tf32} --no-cpu-baseline --no-variants ${OVR:+--override $OVR} 2>&1 | grep -A2 "conv_xn ts" | head -12
done
