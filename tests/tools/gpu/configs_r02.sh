# one bench line per BASELINE config on one B200 (round 2): profiles/r02_configs/<c>.json
mkdir -p gpurun_out/r02_configs
for c in c1 c2 c3 c4 c5b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r02_configs/$c.json 2> gpurun_out/r02_configs/$c.err
done
timeout 900 python bench.py --config c5a --override batch=8 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r02_configs/c5a.json 2> gpurun_out/r02_configs/c5a.err
python - <<'PY'
import json, os
rows = []
for c in ["c1", "c2", "c3", "c4", "c5b", "c5a"]:
    try:
        d = json.loads(open(f"gpurun_out/r02_configs/{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "FAILED", e); continue
    k = d["kernels"]
    fl = k.get("flux_rk", {}).get("hbm_frac", float("nan"))
    pr = k.get("projection", {}).get("hbm_frac", float("nan"))
    ch = k.get("conv_hidden", {}).get("ms_per_launch", 0) * 1e3
    print(f"{c:4s} {d['value']:.4g} cell-upd/s  {d['ms_per_step']:.3f} ms/step  roof {d['roofline']['kernel']} {d['roofline']['frac']:.3f}"
          f"  hidden {ch:.1f} us  flux_hbm {fl:.2f}  proj_hbm {pr:.2f}  e2e {d['e2e']['value']:.4g}  clk {d['clocks']['sm_mhz'] if d['clocks'] else None}")
PY
