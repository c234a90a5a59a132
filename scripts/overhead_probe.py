"""Probe (not product): where the fixed per-launch cost of a streaming kernel goes.

For a device copy, our QuAKE exp and the 512-column softmax at the BASELINE
sizes, time the same rotating-buffer launches two ways:
  evented  — a CUDA event pair around every launch (bench.per_config method);
  batched  — one event pair around R back-to-back launches, divided by R
             (launch i+1 is queued behind launch i, so with PDL its launch
             and prologue overlap launch i's drain).
A 4096-element launch gives the bare launch+completion latency. Run once with
QK_PDL=1 and once with QK_PDL=0.
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
l2 = 126 << 20


def evented(fns, iters=24):
    evs = []
    with torch.cuda.stream(stream):
        for i in range(iters + len(fns)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fns[i % len(fns)]()
            b.record(stream)
            evs.append((a, b))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs[len(fns):]]
    return sum(ts) / len(ts) * 1e3


def batched(fns, reps=6):
    with torch.cuda.stream(stream):
        for f in fns:
            f()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            for f in fns:
                f()
        b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * len(fns))


prm = qk.SoftmaxParams(temperature=0.125)._c()
pdl = os.environ.get("QK_PDL", "1")
for n in (4096, 16 << 20, 25165824, 50331648):
    nbuf = max(2, -(-4 * l2 // (8 * n))) if n > 4096 else 4
    xs = [torch.randn(n, device="cuda") * 2 for _ in range(nbuf)]
    ys = [torch.empty_like(x) for x in xs]
    copy = [lambda x=x, y=y: y.copy_(x) for x, y in zip(xs, ys)]
    ew = [lambda x=x, y=y: L.qk_exp_buffer_device(x.data_ptr(), y.data_ptr(), n, 1, sh)
          for x, y in zip(xs, ys)]
    sm = [lambda x=x, y=y: L.qk_softmax_rows_device(x.data_ptr(), n, 512, ctypes.byref(prm), 1,
                                                     y.data_ptr(), None, sh) for x, y in zip(xs, ys)]
    r = {"pdl": pdl, "n": n, "MB_moved": 8 * n / 1e6, "buffers": nbuf}
    for name, fns in (("copy", copy), ("exp_quake", ew), ("softmax512_quake", sm)):
        e = evented(fns)
        b = batched(fns)
        r[name] = {"evented_us": round(e, 2), "batched_us": round(b, 2),
                   "evented_GBps": round(8 * n / e / 1e3, 1),
                   "batched_GBps": round(8 * n / b / 1e3, 1)}
    print(json.dumps(r), flush=True)
    del xs, ys
    torch.cuda.empty_cache()
