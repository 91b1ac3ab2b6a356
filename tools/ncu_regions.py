"""Share of executed warp instructions per source region of one kernel in an ncu
--set full report (run here, no GPU):
  python tools/ncu_regions.py REP KERNEL_REGEX "{name: (file, first_line, last_line)}"
"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
agg = {}; fname=None; cur=None
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if not r or r[0] == "Line No": continue
    if r[0].isdigit(): cur = (fname, int(r[0]))
    if len(r) > ie and r[2]:
        try: ex = float(r[ie] or 0)
        except ValueError: continue
        agg[cur] = agg.get(cur, 0) + ex
tot = sum(agg.values())
regions = eval(sys.argv[3])
out = {}
for (f, l), v in agg.items():
    name = "other"
    for rn, (rf, a, b) in regions.items():
        if f == rf and a <= l <= b: name = rn; break
    out[name] = out.get(name, 0) + v
print("total warp inst", tot)
for k, v in sorted(out.items(), key=lambda x: -x[1]): print(f"{k:12s} {100*v/tot:5.1f}%  {v/1e6:.1f}M")
