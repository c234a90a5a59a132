"""Probe (not product): a few launches of one elementwise op at its BASELINE size, for
ncu (QK_LIB_PATH selects an alternative build). usage: ew_one.py {logistic|gelu|exp} {1|2}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.workloads import CFG1, CFG2, CFG3  # noqa: E402

op, k = sys.argv[1], int(sys.argv[2])
L = _lib.lib()
w = {"exp": CFG1, "logistic": CFG2, "gelu": CFG3}[op]
x = w.device()
y = torch.empty_like(x)
fn = {"exp": lambda: L.qk_exp_buffer_device(x.data_ptr(), y.data_ptr(), w.n, k, None),
      "logistic": lambda: L.qk_logistic_buffer_device(x.data_ptr(), y.data_ptr(), w.n, k, -1, None),
      "gelu": lambda: L.qk_gelu_buffer_device(x.data_ptr(), y.data_ptr(), w.n, k, -1, None)}[op]
for _ in range(3):
    assert fn() == 0
torch.cuda.synchronize()
