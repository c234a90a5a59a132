"""Tuning sweep (not product): time the cfg5 softmax kernel under different
launch plans (QK_SM_* environment overrides read by plan_softmax)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.workloads import CONFIGS, TUNING  # noqa: E402


def time_plan(w, x, y, env, iters=10):
    for k in ("QK_SM_CLUSTER", "QK_SM_STAGES", "QK_SM_THREADS", "QK_SM_SMEM_KB", "QK_SM_KC",
              "QK_SM_LA"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    L = _lib.lib()
    prm = qk.SoftmaxParams(temperature=w.temperature)._c()
    s = torch.cuda.current_stream().cuda_stream
    kern = int(os.environ.get("SWEEP_KERNEL", "2"))
    fn = lambda: L.qk_softmax_rows_device(x.data_ptr(), w.n, w.cols, ctypes.byref(prm), kern,
                                          y.data_ptr(), None, s)
    for _ in range(3):
        assert fn() == 0, _lib.last_error()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    return ms, qk.softmax_plan(w.cols, True, qk.KernelChoice(kern))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_softmax_vocab"
    if name.startswith("shape:"):  # shape:ROWSxCOLS, N(0, 4)
        from paper_2412_00408_b200.workloads import Workload
        r, c = (int(v) for v in name[6:].split("x"))
        w = Workload(name, "softmax", (r, c), "normal", 0.0, 4.0, 1)
    else:
        w = {**CONFIGS, **TUNING}[name]
    x = w.device()
    y = torch.empty_like(x)
    ref = None
    envs = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}]
    for env in envs:
        try:
            ms, plan = time_plan(w, x, y, env)
        except AssertionError as e:
            print(json.dumps({"env": env, "error": str(e)}))
            continue
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(y.view(-1)[:1000], ref.view(-1)[:1000]))
        gbs = 8 * w.n / (ms * 1e-3) / 1e9
        print(json.dumps({"env": env, "ms": round(ms, 4), "GBps": round(gbs, 1),
                          "plan": {k: plan[k] for k in ("variant", "cluster", "threads", "stages", "slice", "vpt", "resident", "smem")},
                          "first_rows_equal_default": same}), flush=True)


if __name__ == "__main__":
    main()
