"""Top SASS instructions by stall samples and executed count from an ncu
--page source --csv --print-source sass export (run here, no GPU)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
def f(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(f(d["Instructions Executed"]) for d in data)
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(f(d[k]) for d in data) for k in stalls}
print("stall mix:", {k[6:]: round(100 * v / max(tot_s, 1), 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:n]:
    top = sorted(((k[6:], f(d[k])) for k in stalls), key=lambda kv: -kv[1])[:2]
    print(f'{d["Address"]:>6} {100*f(d["Warp Stall Sampling (All Samples)"])/tot_s:5.1f}% ex {f(d["Instructions Executed"]):10.0f} {d["Source"][:60]:60} {top}')
