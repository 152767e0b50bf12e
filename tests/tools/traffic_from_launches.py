"""Per-launch DRAM bytes (read + write) of each kernel class from an ncu launch list -> profiles/ncu_traffic.json.

python tests/tools/traffic_from_launches.py <launches.csv> <config> <precision> <source-note>

Classes follow bench.py's kernel-class names: conv_first / conv_hidden / conv_last (conv_xn_kernel by (CI, CO)),
flux_rk (flux_div_kernel or flux_rk_kernel), projection (the sum of a projection's passes: pen_* kernels per
launch of pen_rows_fwd*, or proj_cluster).
"""
import collections
import csv
import json
import os
import sys

path, cfg, prec, note = sys.argv[1:5]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:]]
per = collections.defaultdict(lambda: collections.defaultdict(float))   # launch id -> metric
names = {}
for d in data:
    key = d["ID"]
    names[key] = d["Kernel Name"]
    if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[key][d["Metric Name"]] += v * scale


def cls(name):
    if "conv_xn_kernel" in name:
        if "<float, 2, 64" in name:
            return "conv_first"
        if "<float, 64, 64" in name:
            return "conv_hidden"
        if "<float, 64, 32" in name:
            return "conv_last"
    if "flux_div" in name or "flux_rk_kernel" in name:
        return "flux_rk"
    if "pen_" in name or "proj_cluster" in name:
        return "projection"
    return None


tot = collections.defaultdict(float)
cnt = collections.defaultdict(int)
for key, m in per.items():
    c = cls(names[key])
    if c is None:
        continue
    tot[c] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    if c != "projection" or "rows_fwd" in names[key] or "proj_cluster" in names[key]:
        cnt[c] += 1
out = {c: tot[c] / cnt[c] for c in tot if cnt[c]}
p = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "profiles", "ncu_traffic.json")
j = json.load(open(p))
j.setdefault(cfg, {})[prec] = out
j[f"_note_{cfg}"] = note
json.dump(j, open(p, "w"), indent=1)
print(json.dumps(out, indent=1))
