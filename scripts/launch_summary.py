"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (evidence aid).

usage: python scripts/launch_summary.py <launches.csv> <out.json> <command>
"""
import csv
import io
import json
import sys
from collections import OrderedDict

src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [l for l in open(src) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
per = OrderedDict()
pipe = []
total = 0.0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1000.0 if r.get("Metric Unit") == "ns" else v * (1000.0 if r.get("Metric Unit") == "ms" else 1.0)
    name = r["Kernel Name"][:80]
    d = per.setdefault(name, {"launches": 0, "total_us": 0.0})
    d["launches"] += 1
    d["total_us"] += us
    total += us
    if "softmax_pipe" in name and us > 300:
        pipe.append(round(us, 1))
for d in per.values():
    d["total_us"] = round(d["total_us"], 1)
    d["share_of_all_gpu_time"] = round(d["total_us"] / total, 4)
json.dump({"command": cmd,
           "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised "
                   "launches. The full-matrix softmax_pipe launches are the device-timed steps (warm-up "
                   "+ timed, 4096 rows each); the shorter ones are the chunked host-span (e2e) path. "
                   "The torch kernels generate the synthetic input / check results outside the timed region.",
           "softmax_pipe_full_matrix_launch_us": pipe, "kernels": per}, open(out, "w"), indent=1)
print(json.dumps({"full_matrix_launch_us": pipe}))
