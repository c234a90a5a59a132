"""Probe (not product): fixed per-launch cost of the cfg5 softmax pipeline.

Times the cfg5-width (128256 cols, QuAKE2) softmax over R rows, R a multiple
of the resident cluster count (every cluster gets R/clusters rows), back to
back and with an event pair per launch; the intercept of a linear fit in
rows-per-cluster is the launch's fixed cost (launch, pipeline fill, drain).
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.workloads import CONFIGS  # noqa: E402

L = _lib.lib()
w = CONFIGS["cfg5_softmax_vocab"]
cols = int(os.environ.get("COLS", w.cols))
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
kern = int(qk.KernelChoice.Quake2)
plan = qk.softmax_plan(cols, True, qk.KernelChoice.Quake2)
res = plan["resident"] or 1
maxrows = (4096 * 128256) // cols
x = (w.device().reshape(-1) if cols == w.cols and os.environ.get("SEEDED") == "1"
     else torch.randn(maxrows * cols, device="cuda") * 4)
y = torch.empty_like(x)
pts = []
extra = [int(v) for v in os.environ.get("ROWS", "").split(",") if v]
for k in (extra or (1, 2, 4, 8, 16, 32, 64, 128)):
    rows = k if extra else res * k
    if rows > maxrows:
        break
    ne = rows * cols

    def f():
        st = L.qk_softmax_rows_device(x.data_ptr(), ne, cols, ctypes.byref(prm), kern,
                                      y.data_ptr(), None, sh)
        assert st == 0, _lib.last_error()

    reps = max(20, 2000 // (rows // res))
    with torch.cuda.stream(stream):
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            f()
        b.record(stream)
        evs = []
        for _ in range(min(reps, 50)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f()
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    b2b = a.elapsed_time(b) * 1e3 / reps
    iso = float(np.mean([e0.elapsed_time(e1) for e0, e1 in evs])) * 1e3
    pts.append((k, b2b, iso))
    print(json.dumps({"cols": cols, "rows": rows, "rows_per_cluster": k, "b2b_us": round(b2b, 2),
                      "isolated_us": round(iso, 2),
                      "b2b_gbps": round(8 * ne / b2b / 1e3, 1)}), flush=True)
if extra:
    sys.exit(0)
ks = np.array([p[0] for p in pts], float)
for j, name in ((1, "b2b"), (2, "isolated")):
    t = np.array([p[j] for p in pts])
    slope, icpt = np.polyfit(ks, t, 1)
    print(json.dumps({"fit": name, "us_per_row_step": round(slope, 3),
                      "fixed_us": round(icpt, 2), "plan": plan}), flush=True)
