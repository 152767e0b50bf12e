# session 5, call 4: persistent four-step passes (N >= 2048): parity + c5a A/B (4 vs 2 columns per CTA)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -x -q -k "projection or slab" > gpurun_out/s5c4_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s5c4_pytest.log
for e in LD_XN_L2EF=0 LD_PEN4_CC2=1; do
  env $e timeout 900 python bench.py --config c5a --override batch=8 --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/s5c4_c5a_$e.json 2> gpurun_out/s5c4_c5a_$e.err
  python - "$e" <<'PY'
import json, sys
e = sys.argv[1]
d = json.loads(open(f"gpurun_out/s5c4_c5a_{e}.json").read().strip().splitlines()[-1])
print("c5a", e, f"{d['value']:.4g}", f"{d['ms_per_step']:.1f} ms/step", {k: (round(v['ms_per_launch'] * 1e3, 1), round(v.get('hbm_frac', 0), 3)) for k, v in d['kernels'].items()})
PY
done
