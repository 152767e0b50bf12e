timeout 200 python tests/tools/tc_quick.py > gpurun_out/tc_quick.log 2>&1; tail -9 gpurun_out/tc_quick.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for p in tf32 f16; do timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline > gpurun_out/bench_$p.log 2>&1; done
python - <<'PY'
import json
for p in ["tf32","f16"]:
    try:
        d=json.loads(open("gpurun_out/bench_%s.log"%p).read().strip().splitlines()[-1])
        print(p, "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], {k:round(v["ms_per_launch"]*1e3,1) for k,v in d["kernels"].items()}, "frac", round(d["roofline"]["frac"],3), "e2e %.3e"%d["e2e"]["value"])
    except Exception as e:
        print(p, "failed", e, open("gpurun_out/bench_%s.log"%p).read()[-2000:])
PY
