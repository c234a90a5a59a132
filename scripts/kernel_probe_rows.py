"""One launch each (after a warm one) of the newer softmax kernels on ~1-2 GB
inputs, for ncu captures: the long-row pipeline (256000 cols), the scalar-lane
pipeline (GPT-2's 50257 cols) and several-rows-per-warp (16 cols)."""
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
for cols, rows in ((256000, 1024), (50257, 5222), (16, 16 << 20)):
    x = torch.randn(rows * cols, device="cuda") * 4
    y = torch.empty_like(x)
    for _ in range(2):
        st = L.qk_softmax_rows_device(x.data_ptr(), rows * cols, cols, ctypes.byref(prm), 2,
                                      y.data_ptr(), None, s)
        assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    print(cols, qk.softmax_plan(cols, cols % 4 == 0, qk.KernelChoice.Quake2))
