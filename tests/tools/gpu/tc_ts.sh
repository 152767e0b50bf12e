timeout 200 python tests/tools/tc_quick.py 2>&1 | tail -9
for d in 8; do
echo "== dbg $d"
LD_NO_GRAPH=1 LD_TC_DEBUG=$d timeout 120 python bench.py --steps 3 --warmup 3 --precision f16 --no-cpu-baseline 2>&1 | grep -A6 "conv_tc ts" | head -7
done
for p in f16 tf32; do timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline > gpurun_out/bench_$p.log 2>&1; done
python - <<'PY'
import json
for p in ["tf32","f16"]:
    d=json.loads(open("gpurun_out/bench_%s.log"%p).read().strip().splitlines()[-1])
    print(p, "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], {k:round(v["ms_per_launch"]*1e3,1) for k,v in d["kernels"].items()}, "frac", round(d["roofline"]["frac"],3), "e2e %.3e"%d["e2e"]["value"])
PY
