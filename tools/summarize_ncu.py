"""Summarises gpurun_out/{launches.csv,full.ncu-rep} into profiles/ (run here, no GPU)."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)

def short(name):
    n = name.split("(")[0]
    for p in ["void ", "svrb::", "<unnamed>::", "(anonymous namespace)::", "unnamed>::"]:
        n = n.replace(p, "")
    return n.strip()

# launch list
rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        agg[short(d["Kernel Name"])].append(float(d["Metric Value"]) / 1000.0)
total = sum(sum(v) for v in agg.values())
lines = [f"# ncu launch list ({tag}): `ncu --metrics gpu__time_duration.sum --clock-control none` "
         f"over tools/profile_step.py (3 config-2 frames, 1024^2, 1,048,573 voxels)", "",
         "| kernel | launches | avg us | share |", "|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/total:.1f}% |")
open(os.path.join(prof, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
os.system(f"cp {os.path.join(OUT, 'launches.csv')} {os.path.join(prof, tag + '_launches.csv')}")

# full capture
rep = os.path.join(OUT, "full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {w: h.index(w) for w in want if w in h}
    units = rr[1]
    per = defaultdict(list)
    for r in rr[2:]:
        if len(r) != len(h):
            continue
        name = short(r[h.index("Kernel Name")])
        per[name].append({w: r[i] for w, i in idx.items()})
    md = [f"# ncu --set full summary ({tag}), warm frame of tools/profile_step.py", "",
          "| kernel | us | DRAM read MB | DRAM write MB | DRAM % | L2 hit % | SM % | issue % | warps active % | regs |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    def f(x):
        try: return float(str(x).replace(",", ""))
        except ValueError: return float("nan")
    for name, lst in per.items():
        d = lst[-1]
        t_us = f(d.get("gpu__time_duration.sum")) / (1000.0 if units[idx["gpu__time_duration.sum"]] == "nsecond" else 1.0)
        unit_r = units[idx["dram__bytes_read.sum"]]
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit_r, 1.0)
        rd = f(d.get("dram__bytes_read.sum")) * scale
        wr = f(d.get("dram__bytes_write.sum")) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units[idx["dram__bytes_write.sum"]], 1.0)
        md.append(f"| {name} | {t_us:.1f} | {rd:.1f} | {wr:.1f} | {f(d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{f(d.get('lts__t_sector_hit_rate.pct')):.1f} | {f(d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{f(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f} | {f(d.get('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | {d.get('launch__registers_per_thread')} |")
        key = {"composite_kernel": "composite", "preprocess_kernel": "preprocess", "onesweep_kernel": "sort",
               "duplicate_kernel": "duplicate"}.get(name.split("<")[0], None)
        if key:
            traffic[key] = (traffic.get(key, 0.0) if key == "sort" else 0.0) + (rd + wr) * 1e6
    open(os.path.join(prof, f"{tag}_ncu_full.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(prof, f"{tag}_launches.md")).read())
if os.path.exists(os.path.join(prof, f"{tag}_ncu_full.md")):
    print(open(os.path.join(prof, f"{tag}_ncu_full.md")).read())
