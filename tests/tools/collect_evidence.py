"""Copy one session's gpurun_out/ evidence into profiles/ (committed text summaries).

python tests/tools/collect_evidence.py <tag> "<note>"      e.g. s6 "round 2 session 6 (final)"

Reads gpurun_out/<tag>_{pytest,smoke,bench}_final.log, <tag>_launches_final.csv, prof_<tag>_final.ncu-rep and
<tag>_configs/*.json; writes profiles/r02_<tag>_*.  Only files that exist are copied.
"""
import json
import os
import subprocess
import sys

tag, note = sys.argv[1], sys.argv[2]
G, P = "gpurun_out", "profiles"
here = os.path.dirname(os.path.abspath(__file__))


def last_json(path):
    for ln in reversed(open(path).read().splitlines()):
        if ln.startswith("{"):
            return json.loads(ln), ln
    return None, None


def tail(path, n):
    return open(path).read().splitlines()[-n:]


# GPU test tail + smoke
pt, sm = f"{G}/{tag}_pytest_final.log", f"{G}/{tag}_smoke_final.log"
if os.path.exists(pt):
    lines = tail(pt, 8) + (tail(sm, 4) if os.path.exists(sm) else [])
    open(f"{P}/r02_{tag}_pytest_gpu_tail.log", "w").write("\n".join(lines) + "\n")
    print(lines[-5] if len(lines) > 4 else lines)

# default bench line
bl = f"{G}/{tag}_bench_final.log"
if os.path.exists(bl):
    d, ln = last_json(bl)
    if d:
        open(f"{P}/r02_{tag}_bench_default.json", "w").write(ln + "\n")
        r = d.get("roofline", {})
        print("bench:", d["value"], d["unit"], d["ms_per_step"], "ms/step; e2e", d["e2e"]["value"],
              "roofline", r.get("bound"), round(r.get("frac", 0), 3), "clocks", d.get("clocks"))

# launch list + traffic
lc = f"{G}/{tag}_launches_final.csv"
if os.path.exists(lc):
    subprocess.check_call([sys.executable, f"{here}/ncu_summary.py", "launches", lc, f"{P}/r02_{tag}_launches_tf32_c4.txt"])
    subprocess.check_call([sys.executable, f"{here}/traffic_from_launches.py", lc, "c4", "tf32",
                           f"c4 TF32, {note} (profiles/r02_{tag}_launches_tf32_c4.txt): per-launch DRAM read + write "
                           "bytes of each kernel class from the ncu launch list of the bench command (ncu flushes "
                           "caches per launch); projection = the sum of one projection's passes"])
rep = f"{G}/prof_{tag}_final.ncu-rep"
if os.path.exists(rep):
    subprocess.check_call([sys.executable, f"{here}/ncu_summary.py", "full", rep, f"{P}/r02_{tag}_ncu_full_c4.txt"])

# per-config table
cd = f"{G}/{tag}_configs"
if os.path.isdir(cd):
    os.makedirs(f"{P}/r02_{tag}_configs", exist_ok=True)
    rows = [f"# {note}: one bench line per BASELINE config on one B200 (bench.py --config c --steps 10 --warmup 3; "
            "c5a: --override batch=8 --steps 3)",
            f"{'cfg':5s} {'cell-upd/s':>10s} {'ms/step':>9s} {'e2e':>10s} {'hidden conv (frac)':>24s} {'out layer':>10s} "
            f"{'flux HBM':>9s} {'proj HBM':>9s} {'clk':>6s}"]
    for c in ("c1", "c2", "c3", "c4", "c5b", "c5a"):
        f = f"{cd}/{c}.json"
        if not os.path.exists(f):
            continue
        d, ln = last_json(f)
        if not d:
            rows.append(f"{c:5s} (no line)")
            continue
        open(f"{P}/r02_{tag}_configs/{c}.json", "w").write(ln + "\n")
        k = d.get("kernels", {})

        def g(name, key, default=float("nan")):
            v = k.get(name, {}).get(key)
            return default if v is None else v
        r = d.get("roofline", {})
        rows.append(f"{c:5s} {d['value']:10.3e} {d['ms_per_step']:9.3f} {d['e2e']['value']:10.3e} "
                    f"{1e3 * g('conv_hidden', 'ms_per_launch'):14.1f} us ({r.get('frac', float('nan')):.2f}) "
                    f"{1e3 * g('conv_last', 'ms_per_launch'):8.1f} us {g('flux_rk', 'hbm_frac'):9.2f} "
                    f"{g('projection', 'hbm_frac'):9.2f} {d.get('clocks', {}).get('sm_mhz', float('nan')):6.0f}")
    open(f"{P}/r02_{tag}_configs/table.txt", "w").write("\n".join(rows) + "\n")
    print("\n".join(rows))
