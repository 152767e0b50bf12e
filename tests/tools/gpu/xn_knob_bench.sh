# conv_xn kernel times (bench events) under LD_XN_DEBUG knobs with a knob build WITHOUT the
# per-role timing instrumentation (no atomics / stamps): clean A/B timings
LD_NVCC_EXTRA="-DLD_XN_KNOBS -DLD_XN_NOTIMING" python -c "from paper_2507_01975_b200 import build as B; B.build(force=True)" || exit 1
for d in ${KNOBS:-0 2 3 4 6 5}; do
  echo -n "dbg=$d  "
  LD_XN_DEBUG=$d bash tests/tools/gpu/variants.sh ${OVR:-""} | cut -c1-200
done
