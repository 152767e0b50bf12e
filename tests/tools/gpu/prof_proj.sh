for p in tf32 f16; do timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline > gpurun_out/bench_$p.log 2>&1; done
python - <<'PY'
import json
for p in ["tf32","f16"]:
    d=json.loads(open("gpurun_out/bench_%s.log"%p).read().strip().splitlines()[-1])
    print(p, "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], {k:round(v["ms_per_launch"]*1e3,1) for k,v in d["kernels"].items()}, "frac", round(d["roofline"]["frac"],3), "e2e %.3e"%d["e2e"]["value"])
PY
bash tests/tools/gpu/ncu_full.sh f16 proj_fused 2 1
