"""Summarises gpurun_out/{launches.csv, full.ncu-rep, bwd.ncu-rep, cfg4.ncu-rep}
into profiles/ (run here, no GPU): per-kernel launch shares and the --set full
metrics, plus profiles/ncu_traffic.json (DRAM bytes per launch of each stage,
per workload) that bench.py reports as roofline.traffic."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
prof = os.environ.get("PROF_DIR", os.path.join(ROOT, "profiles"))
os.makedirs(prof, exist_ok=True)


def short(name):
    n = name.split("(")[0]
    for p in ["void ", "svrb::", "<unnamed>::", "(anonymous namespace)::", "unnamed>::"]:
        n = n.replace(p, "")
    return n.strip()


def f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


# ---- launch list (config 2 frames)
path = os.path.join(OUT, "launches.csv")
if os.path.exists(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    agg = defaultdict(list)
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[short(d["Kernel Name"])].append(f(d["Metric Value"]) / 1000.0)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list ({tag}): `ncu --metrics gpu__time_duration.sum --clock-control none` "
             f"over tools/profile_step.py (3 config-2 frames, 1024^2, 1,048,573 voxels)",
             "", "Cold-cache, serialised launches: compare shares, not absolute times.", "",
             "| kernel | launches | avg us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/total:.1f}% |")
    open(os.path.join(prof, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    os.system(f"cp {path} {os.path.join(prof, tag + '_launches.csv')}")
    print("\n".join(lines))

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0,
         "GB": 1e3}
STAGE = {"composite_kernel": "composite", "composite_coop_kernel": "composite",
         "preprocess_kernel": "preprocess", "onesweep_kernel": "sort",
         "duplicate_packed_kernel": "duplicate", "duplicate_ranked_kernel": "duplicate", "composite_backward_kernel": "backward",
         "voxel_epilogue_kernel": "epilogue", "merge_huge_kernel": "merge"}


def capture(rep_name, title, workload, traffic):
    rep = os.path.join(OUT, rep_name)
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    idx = {w: h.index(w) for w in WANT if w in h}
    per = defaultdict(list)
    for r in rr[2:]:
        if len(r) == len(h):
            per[short(r[h.index("Kernel Name")])].append({w: r[i] for w, i in idx.items()})
    md = [f"# ncu --set full summary ({tag}): {title}", "",
          "| kernel | launches | time us | DRAM read MB | DRAM write MB | DRAM % | L2 hit % | SM % | issue % "
          "| warps active % | regs | warp instr (M) |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    tr = traffic.setdefault(workload, {})
    for name, lst in per.items():
        d = lst[-1]
        t_us = f(d.get("gpu__time_duration.sum")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                                      "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(
            units[idx["gpu__time_duration.sum"]], 1.0)
        rd = f(d.get("dram__bytes_read.sum")) * SCALE.get(units[idx["dram__bytes_read.sum"]], 1.0)
        wr = f(d.get("dram__bytes_write.sum")) * SCALE.get(units[idx["dram__bytes_write.sum"]], 1.0)
        md.append(f"| {name} | {len(lst)} | {t_us:.1f} | {rd:.1f} | {wr:.1f} | "
                  f"{f(d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{f(d.get('lts__t_sector_hit_rate.pct')):.1f} | "
                  f"{f(d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{f(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f} | "
                  f"{f(d.get('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
                  f"{d.get('launch__registers_per_thread')} | {f(d.get('smsp__inst_executed.sum'))/1e6:.1f} |")
        key = STAGE.get(name.split("<")[0])
        if key:  # DRAM bytes per launch (the sort: per onesweep pass, mean over captures)
            if key == "sort":
                bs = [(f(x.get("dram__bytes_read.sum")) * SCALE.get(units[idx["dram__bytes_read.sum"]], 1.0) +
                       f(x.get("dram__bytes_write.sum")) * SCALE.get(units[idx["dram__bytes_write.sum"]], 1.0))
                      for x in lst]
                bs = [b for b in bs if b > 1.0] or bs  # the entries' passes, not the huge-list sort
                tr["sort_pass"] = sum(bs) / len(bs) * 1e6
            else:
                tr[key] = (rd + wr) * 1e6
                tr[key + "_warp_inst"] = f(d.get("smsp__inst_executed.sum"))
    path = os.path.join(prof, f"{tag}_ncu_{rep_name.split('.')[0]}.md")
    open(path, "w").write("\n".join(md) + "\n")
    print("\n".join(md))


traffic = {}
capture("full.ncu-rep", "one warm config-2 frame (tools/profile_step.py)", "cfg2", traffic)
capture("bwd.ncu-rep", "config-3 training step kernels (tools/explore_cfg3.py)", "cfg3", traffic)
capture("cfg4.ncu-rep", "config-4 view 0 (tools/explore_cfg4.py)", "cfg4", traffic)
if "cfg4" in traffic:
    traffic["cfg5"] = dict(traffic["cfg4"])  # same scene and views; backward from cfg3's kernel shape
if "cfg3" in traffic:
    traffic["cfg3i"] = dict(traffic["cfg3"])  # the same view and backward inside the full iteration
if traffic:
    json.dump(traffic, open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
