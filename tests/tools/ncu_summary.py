"""Summarise gpurun_out/ ncu artefacts into profiles/ (text, committed).

python tests/tools/ncu_summary.py launches <launches.csv> <out.txt>
python tests/tools/ncu_summary.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], [dict(zip(rows[0], r)) for r in rows[1:]]
    agg = collections.OrderedDict()
    for d in data:
        k = d["Kernel Name"].split("(")[0][:64]
        agg.setdefault(k, collections.defaultdict(list))[d["Metric Name"]].append(
            float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v.get("gpu__time_duration.sum", [0])) for k, v in agg.items() if not k.startswith("void at::"))
    lines = [f"# ncu launch list ({path}); per-launch device time, cold-cache and serialised (compare shares)",
             f"{'kernel':64s} {'n':>4s} {'t_avg_us':>9s} {'share':>6s} {'dram_rd_MB':>10s} {'dram_wr_MB':>10s}"]
    for k, v in agg.items():
        t = v.get("gpu__time_duration.sum", [0])
        n = len(t)
        share = sum(t) / tot if not k.startswith("void at::") and tot else float("nan")
        lines.append(f"{k:64s} {n:4d} {sum(t) / n / 1e3:9.2f} {share:6.3f} "
                     f"{sum(v.get('dram__bytes_read.sum', [0])) / n / 1e6:10.2f} "
                     f"{sum(v.get('dram__bytes_write.sum', [0])) / n / 1e6:10.2f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {path}"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append("## " + d.get("Kernel Name", "?")[:150])
        for w in WANT:
            if w in d:
                lines.append(f"  {w} = {d[w]} {u.get(w, '')}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
