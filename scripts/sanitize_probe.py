"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family once at small sizes, results checked against the restatement.
Not product code; see scripts/gpu_sanitize.sh."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from oracle.oracle import QUAKE2, Restatement  # noqa: E402
from paper_2412_00408_b200 import lab  # noqa: E402

K = qk.KernelChoice
R = Restatement()
rng = np.random.default_rng(3)
bad = 0
# softmax: warp (512), pipe C=1 (4096, 16384), pipe cluster (50000, 128256), misaligned scalar
for cols, rows in ((512, 16), (4096, 8), (16384, 4), (50000, 3), (128256, 3)):
    for kern in (K.Quake, K.Quake2):
        x = (rng.standard_normal(rows * cols) * 4).astype(np.float32)
        y = qk.softmax_rows(torch.from_numpy(x).cuda(), cols, qk.SoftmaxParams(), kern).cpu().numpy()
        want = R.softmax_rows_ordered(x, cols, qk.softmax_plan(cols, True, kern), 1.0, int(kern))
        bad += int(np.count_nonzero(y.view(np.uint32) != want.view(np.uint32)))
xb = (rng.standard_normal(6 * 517 + 1) * 2).astype(np.float32)
xd = torch.from_numpy(xb).cuda()[1:]
yd = qk.softmax_rows(xd, 517, qk.SoftmaxParams(), K.Quake2).cpu().numpy()
bad += int(np.count_nonzero(yd.view(np.uint32) != R.softmax_rows_ordered(
    xb[1:], 517, qk.softmax_plan(517, False, K.Quake2), 1.0, QUAKE2).view(np.uint32)))
# warp rings: register form (G = 8, 16, 32), three sweeps with agents of 1, 2, 4 and 8 warps;
# aligned and misaligned bases, same and different in/out phases, partial last jobs
for cols, rows in ((197, 37), (257, 21), (513, 13), (1001, 9), (1537, 7), (2049, 11), (4099, 9), (8191, 5)):
    for io, oo in ((0, 0), (1, 1), (2, 3)):
        x = (rng.standard_normal(rows * cols) * 3).astype(np.float32)
        xb = torch.zeros(rows * cols + 4, device="cuda")
        xb[io:io + rows * cols] = torch.from_numpy(x).cuda()
        ob = torch.empty(rows * cols + 4, device="cuda")
        qk.softmax_rows(xb[io:io + rows * cols], cols, qk.SoftmaxParams(), K.Quake2,
                        out=ob[oo:oo + rows * cols])
        want = R.softmax_rows_ordered(x, cols, qk.softmax_plan(cols, False, K.Quake2), 1.0, QUAKE2)
        bad += int(np.count_nonzero(ob[oo:oo + rows * cols].cpu().numpy().view(np.uint32) !=
                                    want.view(np.uint32)))
# elementwise: vector + scalar (misaligned) paths
x = rng.uniform(-100, 100, 100003).astype(np.float32)
for kern in (K.Quake, K.Quake2):
    bad += int(np.count_nonzero(qk.gelu_buffer(x, kern).view(np.uint32) !=
                                R.gelu_buffer(x, int(kern)).view(np.uint32)))
    bad += int(np.count_nonzero(qk.logistic_buffer(x[1:], kern).view(np.uint32) !=
                                R.logistic_buffer(x[1:], int(kern)).view(np.uint32)))
# lab (small)
lab.sweep_error(lab.ExpConfig(K.Quake2, True, False), lab.SweepSpec(-20.0, 20.0, 1 << 16, 64))
lab.continuity_probe(lab.ExpConfig(K.Quake2, False, False), -10, 10)
torch.cuda.synchronize()
print("mismatches", bad)
sys.exit(1 if bad else 0)
