# A/B of measurement env knobs on bench.py lines: ab_env.sh "<config list>" "<VAR=val list>"
# (several variables in one entry: comma-separated, e.g. LD_XN_DEBUG=1,LDSOLVER_LIB=...)
# prints ms/step and per-class us/launch for every (config, env) pair
CFGS=${1:-c4}
ENVS=${2:-"LD_XN_PF=0 LD_XN_PF=1"}
PREC=${PREC:-tf32}
mkdir -p gpurun_out
for c in $CFGS; do for e in $ENVS; do
  t=$(echo "$e" | tr "/=," "___")
  env ${e//,/ } timeout 300 python bench.py --config $c --precision $PREC --steps ${STEPS:-10} --warmup 3 --no-variants --no-cpu-baseline $EXTRA > gpurun_out/ab_${c}_${t}.json 2> gpurun_out/ab_${c}_${t}.err
  python - "$c" "$e" gpurun_out/ab_${c}_${t}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    k = " ".join(f"{n}={v['ms_per_launch']*1e3:.1f}" for n, v in d["kernels"].items())
    print(f"{sys.argv[1]:4s} {sys.argv[2]:22s} ms/step={d['ms_per_step']:.3f} value={d['value']:.4g} clk={d['clocks']['sm_mhz'] if d['clocks'] else None} | {k}")
except Exception as ex:
    print(sys.argv[1], sys.argv[2], "FAILED", ex)
PY
done; done
