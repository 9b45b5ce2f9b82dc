mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e > gpurun_out/launches.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_series_stats -s 1 -c 1 -f -o gpurun_out/prof_stats python tools/profile_run.py 2 > gpurun_out/prof_stats.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open("gpurun_out/launches.csv") if not l.startswith("==")))
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"][:60]; m = r["Metric Name"]; v = float(r["Metric Value"].replace(",", ""))
    agg.setdefault(k, collections.defaultdict(list))[m].append(v)
for k, d in agg.items():
    t = d["gpu__time_duration.sum"]
    print(f"{k:60s} n={len(t):4d} mean_us={sum(t)/len(t)/1e3:8.2f} rd_MB={sum(d['dram__bytes_read.sum'])/len(t)/1e6:8.1f}")
PY
