"""Per-SASS-instruction executed counts of an ncu report (tuning aid, not product).

usage: python scripts/ncu_inst_sass.py <report.ncu-rep> <out.txt>
Reads `ncu -i --page source --csv --print-source sass` and writes every SASS
line with its warp-level executed count, plus the total.
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r:
        hdr, body = r, rows[i + 1:]
        break
if hdr is None:
    open(out, "w").write("no source page\n" + txt[:2000])
    sys.exit(0)
cands = [c for c in hdr if "Instructions Executed" in c]
col = [c for c in cands if "Thread" not in c and "Predicated" not in c]
ci = hdr.index(col[0] if col else cands[0])
src = hdr.index("Source")


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


total = sum(num(r[ci]) for r in body if len(r) > ci)
with open(out, "w") as f:
    f.write(f"columns: {cands}; using {hdr[ci]}; total {total:.0f}\n")
    for r in body:
        if len(r) > ci:
            f.write(f"{num(r[ci]):12.0f}  {r[src]}\n")
