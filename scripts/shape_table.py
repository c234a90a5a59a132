"""Markdown table (softmax by row length) from a softmax_shape_sweep.py log.
usage: python scripts/shape_table.py profiles/r02_softmax_shape_sweep.jsonl"""
import json
import sys

print("| cols | aligned | kernel | lanes / CTA threads | cluster | GB/s | frac |")
print("|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    r = json.loads(line)
    name = {"ring": "wring"}.get(r["kernel"], r["kernel"])
    print(f"| {r['cols']} | {'yes' if r['aligned'] else 'no'} | `{name}` | {r['lanes']} / {r.get('threads', '')} | "
          f"{r['cluster']} | {r['gbps']:.0f} | {r['frac']:.2f} |")
