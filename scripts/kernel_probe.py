"""One launch each of the cfg2 logistic QuAKE2, cfg3 GELU QuAKE2 and cfg4
softmax QuAKE2 kernels (device API; cfg4 runs softmax_subwarp), for ncu captures."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.workloads import CFG2, CFG3, CFG4  # noqa: E402

L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
for w in (CFG2, CFG3, CFG4):
    x = w.device()
    y = torch.empty_like(x)
    for _ in range(2):
        if w.op == "logistic":
            st = L.qk_logistic_buffer_device(x.data_ptr(), y.data_ptr(), w.n, 2, -1, s)
        elif w.op == "gelu":
            st = L.qk_gelu_buffer_device(x.data_ptr(), y.data_ptr(), w.n, 2, -1, s)
        else:
            prm = qk.SoftmaxParams(temperature=w.temperature)._c()
            st = L.qk_softmax_rows_device(x.data_ptr(), w.n, w.cols, ctypes.byref(prm), 2,
                                          y.data_ptr(), None, s)
        assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
print("ok")
