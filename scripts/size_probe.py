"""Probe (not product): steady-state time of a copy, our elementwise exp and the
512-column softmax at the same sizes, rotating buffers >= 4x L2 (bench.per_config
method). Shows whether the softmax has headroom below the streaming ceiling."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

L = _lib.lib()
K = qk.KernelChoice
stream = torch.cuda.Stream()
sh = stream.cuda_stream
l2 = 126 << 20


def timeit(fns, iters=24):
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


prm = qk.SoftmaxParams(temperature=0.125)._c()
for n in (16 << 20, 25165824, 50331648, 100663296):
    nbuf = max(2, -(-4 * l2 // (8 * n)))
    xs = [torch.randn(n, device="cuda") * 2 for _ in range(nbuf)]
    ys = [torch.empty_like(x) for x in xs]
    copy = [lambda x=x, y=y: y.copy_(x) for x, y in zip(xs, ys)]
    ew = [lambda x=x, y=y: L.qk_exp_buffer_device(x.data_ptr(), y.data_ptr(), n, 1, sh)
          for x, y in zip(xs, ys)]
    sm = [lambda x=x, y=y: L.qk_softmax_rows_device(x.data_ptr(), n, 512, ctypes.byref(prm), 1,
                                                     y.data_ptr(), None, sh) for x, y in zip(xs, ys)]
    r = {"n": n, "MB_moved": 8 * n / 1e6}
    for name, fns in (("copy", copy), ("exp_quake", ew), ("softmax512_quake", sm)):
        us = timeit(fns)
        r[name] = {"us": round(us, 2), "GBps": round(8 * n / us / 1e3, 1)}
    print(json.dumps(r), flush=True)
    del xs, ys
