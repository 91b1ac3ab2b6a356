"""Per-kernel average duration from an ncu --metrics gpu__time_duration.sum CSV
(cold-cache, serialised launches: compare shares, not absolute times).
usage: python tools/kernel_times.py gpurun_out/x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
agg = defaultdict(list)
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] == "gpu__time_duration.sum":
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d.get("Metric Unit", "nsecond"), 1e-3)
        agg[d["Kernel Name"].split("(")[0].replace("void ", "").replace("svrb::", "")
            .replace("<unnamed>::", "")].append(float(d["Metric Value"].replace(",", "")) * scale)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):4d} avg={sum(v)/len(v):9.1f} us")
