"""Summarise an ncu report (--set full) into a small committed JSON/markdown.

usage: python scripts/ncu_summary.py <report.ncu-rep> <out_prefix> [label]
writes <out_prefix>.json and <out_prefix>.md with, per profiled kernel:
duration, DRAM bytes read/write (the `traffic` figure bench.py reports),
DRAM throughput %, IPC, issue-slot busy %, registers, occupancy, grid/cluster
shape, top stall reasons and the instruction mix.
"""
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units = raw[0], raw[1]
    kernels = []
    for row in raw[2:]:
        d = dict(zip(hdr, row))

        def f(k):
            try:
                return float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return None

        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        stalls = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda t: -t[1])[:8])
        pipes = {k.split("pipe_")[1].split(".")[0]: f(k) for k in d
                 if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")}
        kernels.append({
            "kernel": d.get("Kernel Name"),
            "duration": f("gpu__time_duration.sum"),
            "duration_unit": units[hdr.index("gpu__time_duration.sum")],
            "dram_bytes_read": f("dram__bytes_read.sum"),
            "dram_bytes_write": f("dram__bytes_write.sum"),
            "dram_unit": units[hdr.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in hdr else None,
            "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "ipc_active": f("sm__inst_executed.avg.per_cycle_active"),
            "issue_busy_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "inst_executed": f("smsp__inst_executed.sum"),
            "registers": f("launch__registers_per_thread"),
            "block": f("launch__block_size"),
            "grid": f("launch__grid_size"),
            "cluster": f("launch__cluster_size") if "launch__cluster_size" in hdr else None,
            "smem_dynamic": f("launch__shared_mem_per_block_dynamic"),
            "achieved_warps_per_sm": f("sm__warps_active.avg.per_cycle_active"),
            "sm_clock": f("smsp__cycles_elapsed.avg.per_second"),
            "sm_clock_unit": units[hdr.index("smsp__cycles_elapsed.avg.per_second")]
            if "smsp__cycles_elapsed.avg.per_second" in hdr else None,
            "top_stalls": stalls,
            "pipe_util_pct": {k: v for k, v in pipes.items() if v},
        })
    with open(prefix + ".json", "w") as fh:
        json.dump({"report": rep, "label": label, "kernels": kernels}, fh, indent=1)
    with open(prefix + ".md", "w") as fh:
        fh.write(f"# ncu summary {label}\n\nsource: `{rep}` (--set full --clock-control none)\n\n")
        for k in kernels:
            fh.write(f"## {k['kernel'][:120]}\n\n")
            for key in ("duration", "duration_unit", "dram_bytes_read", "dram_bytes_write", "dram_unit",
                        "dram_throughput_pct", "ipc_active", "issue_busy_pct", "inst_executed",
                        "registers", "block", "grid", "cluster", "smem_dynamic",
                        "achieved_warps_per_sm", "sm_clock", "sm_clock_unit"):
                fh.write(f"- {key}: {k[key]}\n")
            fh.write(f"- top stalls (samples): {k['top_stalls']}\n")
            fh.write(f"- pipe utilisation %: {k['pipe_util_pct']}\n\n")
    print(json.dumps(kernels, indent=1)[:2000])


if __name__ == "__main__":
    main()
