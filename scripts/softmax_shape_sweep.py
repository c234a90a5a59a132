"""Probe (not product): the softmax planner's choice and back-to-back throughput
for representative row lengths (aligned and not), ~4.2 GB moved per launch,
QuAKE2, N(0, 4) inputs."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

NAMES = {1: "warp_scalar", 2: "smem", 3: "global3", 4: "pipe", 6: "pipe_l2", 7: "pipe_s",
         9: "thread_row", 10: "rows_smem", 11: "subwarp", 12: "tiles", 13: "span", 14: "ring"}
# IOFF / OOFF: input / output offsets in floats (0-3) from a 16-byte boundary
IOFF, OOFF = int(os.environ.get("IOFF", "0")), int(os.environ.get("OOFF", "0"))
L = _lib.lib()
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
total = 4096 * 128256
xb = torch.randn(total + 4, device="cuda") * 4
yb = torch.empty_like(xb)
x, y = xb[IOFF:IOFF + total], yb[OOFF:OOFF + total]
cols_list = [int(c) for c in os.environ.get("COLS", "4,7,16,31,32,64,77,127,128,197,256,257,512,"
                                            "577,1001,1024,2047,4096,4097,16384,50000,50257,"
                                            "128256,151936,151937,202048,256000,262144").split(",")]
for cols in cols_list:
    time.sleep(float(os.environ.get("SLEEP", "1.0")))  # let the clocks recover between shapes
    rows = total // cols
    n = rows * cols
    plan = qk.softmax_plan(cols, cols % 4 == 0, qk.KernelChoice.Quake2)

    def f():
        st = L.qk_softmax_rows_device(x.data_ptr(), n, cols, ctypes.byref(prm), 2, y.data_ptr(),
                                      None, sh)
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
    gbs = 8 * n / us / 1e3
    print(json.dumps({"cols": cols, "aligned": cols % 4 == 0, "ioff": IOFF, "ooff": OOFF,
                      "kernel": NAMES[plan["variant"]],
                      "lanes": plan["lanes"], "cluster": plan["cluster"], "threads": plan["threads"],
                      "stages": plan["stages"], "smem": plan["smem"], "us": round(us, 1),
                      "gbps": round(gbs, 1), "frac": round(gbs / peak, 3)}), flush=True)
