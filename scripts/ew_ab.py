"""Probe (not product): back-to-back time of the cfg1/cfg2/cfg3 elementwise kernels for
the library QK_LIB_PATH points at (A/B of two builds), rotating buffers >= 4x L2."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_00408_b200 import _lib  # noqa: E402

L = _lib.lib()
stream = torch.cuda.Stream()
sh = stream.cuda_stream
l2 = 126 << 20
res = {}
for name, n, fn, extra in (("exp", 1 << 24, L.qk_exp_buffer_device, ()),
                           ("logistic", 1 << 24, L.qk_logistic_buffer_device, (-1,)),
                           ("gelu", 16384 * 3072, L.qk_gelu_buffer_device, (-1,))):
    pairs = max(2, -(-4 * l2 // (8 * n)))
    xs = [torch.randn(n, device="cuda") for _ in range(pairs)]
    ys = [torch.empty_like(x) for x in xs]
    for k in (1, 2):
        fns = [lambda x=x, y=y: fn(x.data_ptr(), y.data_ptr(), n, k, *extra, sh) for x, y in zip(xs, ys)]
        with torch.cuda.stream(stream):
            for f in fns:
                f()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(8):
                for f in fns:
                    f()
            b.record(stream)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (8 * pairs)
        res[f"{name}:k{k}"] = round(us, 2)
    del xs, ys
print(json.dumps({"lib": os.environ.get("QK_LIB_PATH", "default"), **res}))
