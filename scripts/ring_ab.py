"""Probe (not product): A/B of softmax planner option sets on the same rows,
interleaved in one process (ABAB...) so both see the same clocks. ~4.2 GB moved
per launch, QuAKE2 (KERNEL=1 for QuAKE), N(0, 4) inputs.
MODES: ';'-separated option sets, each 'NAME=V,NAME=V' ('' = the defaults)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

NAMES = {1: "warp_scalar", 2: "smem", 3: "global3", 4: "pipe", 6: "pipe_l2", 7: "pipe_s",
         9: "thread_row", 10: "rows_smem", 11: "subwarp", 12: "tiles", 13: "span", 14: "ring"}
L = _lib.lib()
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
KERN = int(os.environ.get("KERNEL", "2"))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
total = int(os.environ.get("TOTAL", str(4096 * 128256)))
x = torch.randn(total, device="cuda") * 4
y = torch.empty_like(x)
modes = [m for m in os.environ.get("MODES", ";QK_SM_RING=1").split(";")]
cols_list = [int(c) for c in os.environ["COLS"].split(",")]
REPS, ITERS = int(os.environ.get("REPS", "3")), int(os.environ.get("ITERS", "8"))


def apply(mode):
    for kv in filter(None, mode.split(",")):
        k, v = kv.split("=")
        qk.set_plan_override(k, int(v))


def clear(mode):
    for kv in filter(None, mode.split(",")):
        qk.set_plan_override(kv.split("=")[0], 0, clear=True)


for cols in cols_list:
    rows = total // cols
    n = rows * cols
    best = {}
    plans = {}
    for rep in range(REPS):
        for mode in modes:
            apply(mode)
            plan = qk.softmax_plan(cols, True, qk.KernelChoice(KERN))
            plans[mode] = plan

            def f():
                st = L.qk_softmax_rows_device(x.data_ptr(), n, cols, ctypes.byref(prm), KERN,
                                              y.data_ptr(), None, sh)
                assert st == 0, _lib.last_error()

            with torch.cuda.stream(stream):
                for _ in range(2):
                    f()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(ITERS):
                    f()
                b.record(stream)
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / ITERS
            best.setdefault(mode, []).append(us)
            clear(mode)
    out = {"cols": cols}
    for mode in modes:
        us = sorted(best[mode])[len(best[mode]) // 2]
        pl = plans[mode]
        out[mode or "default"] = {"kernel": NAMES[pl["variant"]], "lanes": pl["lanes"], "vpt": pl["vpt"],
                                  "threads": pl["threads"], "stages": pl["stages"],
                                  "us": round(us, 1), "frac": round(8 * n / us / 1e3 / peak, 3)}
    print(json.dumps(out), flush=True)
