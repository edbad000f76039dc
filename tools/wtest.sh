python -m pytest tests -m gpu -x -q -k "wasserstein or block_means or timeseries" > gpurun_out/t_w.log 2>&1; tail -2 gpurun_out/t_w.log
QB_OPS=wasserstein python tools/quick_bench.py c2 c3 c5 2>&1 | grep -E "==|wasser"
QB_OPS=wasserstein timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wass_launches.csv python tools/quick_bench.py c3 > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/wass_launches.csv")) if len(r)>10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
agg=collections.OrderedDict()
for r in rows[1:]:
    n=r[ix["Kernel Name"]].split("(")[0]; v=float(r[ix["Metric Value"]].replace(",",""))/1000
    a=agg.setdefault(n,[0,0.0]); a[0]+=1; a[1]+=v
for n,(c,t) in agg.items(): print(f"{n[:40]:40s} {c:4d} {t:9.1f} us")
PY
