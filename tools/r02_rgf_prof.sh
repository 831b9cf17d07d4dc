#!/bin/bash
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_rgf_launches.csv python tools/rgf_time.py rgf_finfet 1 > gpurun_out/r02_rgf_ncu.log 2>&1
echo rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/r02_rgf_launches.csv")))
h = None
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows:
    if r and r[0] == "ID": h = r; continue
    if h is None or len(r) != len(h): continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    ms = v / 1e6 if unit == "nsecond" else v / 1e3 if unit == "usecond" else v
    agg[d["Kernel Name"][:90]][0] += ms; agg[d["Kernel Name"][:90]][1] += 1
for k, (ms, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:15]:
    print(f"{ms:10.1f} ms {n:6d}  {k}")
PY
