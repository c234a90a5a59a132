"""One launch each (after a warm one) of the short-row softmax kernels (128 and
64 aligned columns, ~1 GB), for ncu captures."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402

L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
prm = qk.SoftmaxParams(temperature=1.0)._c()
for cols in (128, 64):
    rows = (1 << 28) // cols
    x = torch.randn(rows * cols, device="cuda") * 4
    y = torch.empty_like(x)
    for _ in range(2):
        st = L.qk_softmax_rows_device(x.data_ptr(), rows * cols, cols, ctypes.byref(prm), 2,
                                      y.data_ptr(), None, s)
        assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    print(cols, qk.softmax_plan(cols, True, qk.KernelChoice.Quake2))
