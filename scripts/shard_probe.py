"""Probe (not product): the per-rank work of the row-sharded cfg5 run, on one GPU.

Under `torchrun --nproc-per-node N bench.py` rank r softmaxes rows
shard.row_shard(4096, r, N) of cfg5 on its own GPU with no collective, so the
job time is the slowest rank's kernel time. This box has one GPU: time rank
0's shard (the largest; shards differ by at most one row) back to back, and
report what each rank does and the aggregate it implies if every GPU runs its
shard as fast as this one. Row-granular persistent scheduling caps a rank at
rows / (resident clusters * ceil(rows / resident clusters)).
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.shard import row_shard  # noqa: E402
from paper_2412_00408_b200.workloads import CONFIGS  # noqa: E402

L = _lib.lib()
w = CONFIGS["cfg5_softmax_vocab"]
stream = torch.cuda.Stream()
sh = stream.cuda_stream
prm = qk.SoftmaxParams(temperature=w.temperature)._c()
kern = int(qk.KernelChoice.Quake2)
plan = qk.softmax_plan(w.cols, True, qk.KernelChoice.Quake2)
x = w.device()
y = torch.empty_like(x)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
for n in (1, 2, 4, 8):
    r0, r1 = row_shard(w.rows, 0, n)
    rows = r1 - r0
    xs, ys = x[r0:r1], y[r0:r1]
    ne = rows * w.cols

    def f():
        st = L.qk_softmax_rows_device(xs.data_ptr(), ne, w.cols, ctypes.byref(prm), kern,
                                      ys.data_ptr(), None, sh)
        assert st == 0, _lib.last_error()

    reps = 40
    with torch.cuda.stream(stream):
        for _ in range(3):
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            f()
        b.record(stream)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    res = plan["resident"]
    cap = rows / (res * -(-rows // res)) if res else None
    gbs = 8 * ne / us / 1e3
    print(json.dumps({"gpus": n, "rows_per_rank": rows, "rank_us": round(us, 2),
                      "rank_gbps": round(gbs, 1), "rank_frac": round(gbs / peak, 4),
                      "row_balance_cap": round(cap, 4) if cap else None,
                      "implied_job_elements_per_s": w.n / (us * 1e-6),
                      "resident_clusters": res}), flush=True)
