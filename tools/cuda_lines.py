"""Per-CUDA-line instructions executed + stall samples from
`ncu -i X --page source --csv --print-source cuda,sass` (run here, no GPU)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
fname, out = None, []
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]
    elif r and r[0] not in ("", "Line No", "Function Name") and len(r) > ie:
        try: out.append((float(r[ie] or 0), float(r[ws] or 0), fname, r[0], r[1].strip()[:80]))
        except ValueError: pass
tot = sum(o[0] for o in out); tots = sum(o[1] for o in out)
print(f"total warp instructions {tot:.4e}, samples {tots:.0f}")
for ex, s, f, ln, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*ex/tot:5.1f}% {100*s/tots:5.1f}%s {f}:{ln:5} {src}")
