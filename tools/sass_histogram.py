"""SASS opcode histograms (no GPU):
    python tools/sass_histogram.py paper_2412_04459_b200/build/raster.o REGEX [REGEX ...]   (static)
    python tools/sass_histogram.py --ncu REP.ncu-rep KERNEL_REGEX                            (executed)
Counts instructions per opcode (modifiers dropped) and flags the Blackwell
memory paths (LDGSTS = cp.async, UTMALDG/UBLKCP = TMA, REDG/RED = reductions)."""
import collections
import re
import subprocess
import sys

def static(obj, pats):
  sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
  funcs = re.split(r"\n\s*Function : ", sass)
  for pat in pats:
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not re.search(pat, name):
            continue
        ops = collections.Counter()
        for line in f.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(2)] += 1
        table(f"`{name}` (static)", ops)


def table(title, ops, top=40):
    total = sum(ops.values()) or 1
    print(f"## {title}\n\n{total:.0f} instructions\n")
    print("| opcode | count | share |\n|---|---|---|")
    for op, c in ops.most_common(top):
        print(f"| {op} | {c:.0f} | {100 * c / total:.1f}% |")
    print()


def executed(rep, kern):
    """Executed-instruction histogram per opcode from an ncu --set full report."""
    import csv
    import io
    raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if r and "Source" in r and "Instructions Executed" in r)
    src, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    ops = collections.Counter()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= ie or not r[ie]:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[src])
        try:
            if m:
                ops[m.group(2)] += float(r[ie])
        except ValueError:
            pass
    return ops


if __name__ == "__main__":
    if sys.argv[1] == "--ncu":  # --ncu REP KERNEL_REGEX
        table(f"`{sys.argv[3]}` (executed, {sys.argv[2].split('/')[-1]})", executed(sys.argv[2], sys.argv[3]))
    else:
        static(sys.argv[1], sys.argv[2:])
