# one bench line per BASELINE config (single GPU), kernel shares and HBM fractions
for c in ${CONFIGS:-c1 c2 c3 c4 c5b}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-variants ${EXTRA} > gpurun_out/cfg_$c.log 2>&1
  tail -1 gpurun_out/cfg_$c.log > gpurun_out/cfg_$c.json
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/cfg_$c.json").read())
    print("$c", "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], "frac %.3f"%d["roofline"]["frac"],
          {k:(round(v["ms_per_launch"]*1e3,1), round(v.get("hbm_frac",0),2)) for k,v in d["kernels"].items()})
except Exception as e:
    print("$c failed", e, open("gpurun_out/cfg_$c.log").read()[-600:])
PY
done
