"""Probe (not product): the long-row pipeline (kPipeL2, QK_SM_L2=1) vs the default plan.

For each row length: bit-exactness of kPipeL2 against the ordered restatement
on a few rows (the checker, oracle/), then back-to-back timings (~4.2 GB per
launch) of the default plan and of kPipeL2 at each cluster size / prefetch
distance.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from oracle.oracle import QUAKE2, Restatement  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

L = _lib.lib()
R = Restatement()
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
kern = int(qk.KernelChoice.Quake2)
cols_list = [int(c) for c in os.environ.get("COLS", "128256,151936,202048,256000,262144,300000").split(",")]
clusters = [int(c) for c in os.environ.get("CLUSTERS", "0").split(",")]  # 0 = planner's choice
pfs = [int(c) for c in os.environ.get("PFS", "2").split(",")]


def env(**kw):
    for k in ("QK_SM_L2", "QK_SM_CLUSTER", "QK_SM_PF"):
        os.environ.pop(k, None)
    for k, v in kw.items():
        os.environ[k] = str(v)


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
    return us, 8 * ne / us / 1e3


for cols in cols_list:
    rows = 4096 * 128256 // cols
    x = torch.randn(rows * cols, device="cuda") * 4
    y = torch.empty_like(x)
    env()
    plan = qk.softmax_plan(cols, True, qk.KernelChoice.Quake2)
    us, gbs = run(cols, x, y, rows)
    print(json.dumps({"cols": cols, "mode": "default", "us": round(us, 1), "gbps": round(gbs, 1),
                      "plan": plan}), flush=True)
    for c in clusters:
        for pf in pfs:
            kw = {"QK_SM_L2": 1, "QK_SM_PF": pf}
            if c:
                kw["QK_SM_CLUSTER"] = c
            env(**kw)
            plan = qk.softmax_plan(cols, True, qk.KernelChoice.Quake2)
            if plan["variant"] != 6:
                print(json.dumps({"cols": cols, "mode": f"l2 C={c}", "skipped": plan}), flush=True)
                continue
            # parity on a few rows against the ordered restatement of this plan
            nr = 8
            xs = x[: nr * cols]
            ys = torch.empty_like(xs)
            st = L.qk_softmax_rows_device(xs.data_ptr(), nr * cols, cols, ctypes.byref(prm), kern,
                                          ys.data_ptr(), None, sh)
            assert st == 0, _lib.last_error()
            torch.cuda.synchronize()
            want = R.softmax_rows_ordered(xs.cpu().numpy(), cols, plan, 1.0, QUAKE2)
            exact = bool(np.array_equal(ys.cpu().numpy().view(np.uint32), want.view(np.uint32)))
            us, gbs = run(cols, x, y, rows)
            print(json.dumps({"cols": cols, "mode": f"l2 C={plan['cluster']} pf={pf}",
                              "us": round(us, 1), "gbps": round(gbs, 1), "bitexact": exact,
                              "plan": plan}), flush=True)
    del x, y
    torch.cuda.empty_cache()
