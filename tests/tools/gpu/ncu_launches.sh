# per-launch device times of one bench run (ncu serialises launches; compare shares)
P=${1:-f16}
python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline > gpurun_out/plain_$P.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 1 --precision $P --no-cpu-baseline > gpurun_out/ncu_launch_$P.log 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/launches_$P.csv")) if len(r)>10]
hdr=rows[0]; data=[dict(zip(hdr,r)) for r in rows[1:]]
agg=collections.OrderedDict()
for d in data:
    k=d["Kernel Name"][:60]; m=d["Metric Name"]; v=float(d["Metric Value"].replace(",",""))
    agg.setdefault(k,collections.defaultdict(list))[m].append(v)
for k,v in agg.items():
    t=v.get("gpu__time_duration.sum",[0])
    print("%-60s n=%3d t_avg=%8.2f us rd=%7.1f MB wr=%7.1f MB sm%%=%5.1f"%(k,len(t),sum(t)/len(t)/1e3,
        sum(v.get("dram__bytes_read.sum",[0]))/len(t)/1e6, sum(v.get("dram__bytes_write.sum",[0]))/len(t)/1e6,
        sum(v.get("sm__throughput.avg.pct_of_peak_sustained_elapsed",[0]))/len(t)))
PY
