# launch times of the large-N spectral passes (O_F at c4, history TC at c4) -- measurement only
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-variants"
for tag in "fno:fno_kmax=12,fno_layers=2,fno_width=8" "tch:tc_head=0,tc_mode=1,tc_interval=4,tc_kmax=12,tc_layers=2,tc_width=8"; do
  name=${tag%%:*}; ov=${tag#*:}
  LD_HOST_NO_PIPELINE=1 timeout 600 ncu --kernel-name regex:"spec_big|hist|push" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 40 --csv --log-file gpurun_out/r02_ncu_big_$name.csv $B --override $ov > /dev/null 2>&1
  python - "$name" <<'PY'
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(f"gpurun_out/r02_ncu_big_{sys.argv[1]}.csv") if l.startswith('"')))
agg = collections.defaultdict(list)
for r in rows:
    agg[(r["Kernel Name"][:40], r["Metric Name"])].append(float(r["Metric Value"].replace(",", "")))
for (k, m), v in sorted(agg.items()):
    print(sys.argv[1], k, m, len(v), sum(v) / len(v))
PY
done
