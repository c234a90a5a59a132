"""Probe (not product): two-stage vs single-stage softmax pipelines on long rows.

For each row length, times (back to back, ~4.2 GB moved per launch) the
planner's default plan and the single-stage schedule (QK_SM_STAGES=1) at each
feasible cluster size, and checks every row sums to 1 within 1e-4.

The single-stage schedule was measured with this script, rejected
(profiles/r01_single_stage_long_rows.jsonl) and removed from
the kernel; QK_SM_STAGES=1 now leaves only the default rows.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

L = _lib.lib()
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
kern = int(qk.KernelChoice.Quake2)
cols_list = [int(c) for c in os.environ.get("COLS", "151936,202048,256000,262144,300000").split(",")]
clusters = [int(c) for c in os.environ.get("CLUSTERS", "4,5,6,7,8,9,10,11,12").split(",")]


def run(cols, x, y, rows):
    ne = rows * cols

    def f():
        st = L.qk_softmax_rows_device(x.data_ptr(), ne, cols, ctypes.byref(prm), kern,
                                      y.data_ptr(), None, sh)
        assert st == 0, _lib.last_error()

    with torch.cuda.stream(stream):
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            f()
        b.record(stream)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 10
    s = y[:ne].view(rows, cols).double().sum(1)
    ok = bool(((s - 1).abs() < 1e-4).all())
    return us, 8 * ne / us / 1e3, ok


for cols in cols_list:
    rows = 4096 * 128256 // cols
    x = torch.randn(rows * cols, device="cuda") * 4
    y = torch.empty_like(x)
    for k in ("QK_SM_STAGES", "QK_SM_CLUSTER"):
        os.environ.pop(k, None)
    plan = qk.softmax_plan(cols, True, qk.KernelChoice.Quake2)
    us, gbs, ok = run(cols, x, y, rows)
    print(json.dumps({"cols": cols, "rows": rows, "mode": "default", "us": round(us, 1),
                      "gbps": round(gbs, 1), "sums_ok": ok, "plan": plan}), flush=True)
    os.environ["QK_SM_STAGES"] = "1"
    for c in clusters:
        os.environ["QK_SM_CLUSTER"] = str(c)
        plan = qk.softmax_plan(cols, True, qk.KernelChoice.Quake2)
        if plan["variant"] != 4 or plan["cluster"] != c:
            continue
        us, gbs, ok = run(cols, x, y, rows)
        print(json.dumps({"cols": cols, "rows": rows, "mode": f"single C={c}", "us": round(us, 1),
                          "gbps": round(gbs, 1), "sums_ok": ok, "plan": plan}), flush=True)
    del x, y
    torch.cuda.empty_cache()
