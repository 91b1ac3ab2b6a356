"""Per-source-line instruction and stall-sample shares of one kernel in an
ncu --set full report (run here, no GPU):
python tools/hotspots.py gpurun_out/full.ncu-rep composite_kernel 30"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg, cur, fname = {}, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if not r or r[0] == "Line No":
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:90])
    if len(r) > ie and r[2]:
        try:
            ex, st = float(r[ie] or 0), float(r[ws] or 0)
        except ValueError:
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += ex
        a[1] += st
tot = sum(v[0] for v in agg.values()) or 1.0
tots = sum(v[1] for v in agg.values()) or 1.0
print(f"| instr % | stall % | line | source |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"| {100 * v[0] / tot:.1f} | {100 * v[1] / tots:.1f} | {k[0]}:{k[1]} | `{k[2]}` |")
