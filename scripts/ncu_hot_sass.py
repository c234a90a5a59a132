"""Top SASS instructions of an ncu report by stall samples (tuning aid, not product).

usage: python scripts/ncu_hot_sass.py <report.ncu-rep> <out.txt> [N]
Reads `ncu -i --page source --csv --print-source sass` and keeps the N lines
with the most warp-stall samples, with their stall-reason columns.
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 60
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and any("Sampling" in c for c in r):
        hdr, body = r, rows[i + 1:]
        break
if hdr is None:
    open(out, "w").write("no source page\n" + txt[:2000])
    sys.exit(0)
samp = [c for c in hdr if c.startswith("Warp Stall Sampling (All")][0]
si = hdr.index(samp)
src = hdr.index("Source")
addr = hdr.index("Address") if "Address" in hdr else 0
stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") or "Stall" in c and i != si]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


total = sum(num(r[si]) for r in body if len(r) > si)
top = sorted((r for r in body if len(r) > si), key=lambda r: -num(r[si]))[:n]
with open(out, "w") as f:
    f.write(f"total samples {total:.0f}; columns: {samp}\n")
    for r in top:
        f.write(f"{num(r[si]):8.0f} {100 * num(r[si]) / max(total, 1):5.1f}%  {r[addr]:>8}  {r[src]}\n")
    # whole-kernel listing, compact: address, samples, instruction
    f.write("\n--- full listing ---\n")
    for r in body:
        if len(r) > si:
            f.write(f"{r[addr]:>8} {num(r[si]):7.0f}  {r[src]}\n")
