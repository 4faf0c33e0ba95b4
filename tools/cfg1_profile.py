"""cfg1 (2048^2, d = 3): where a public-API solve spends its time.

Prints, for the 100-iteration fixed solve and the tolerance solve:
  * the bench step (CUDA events on torch's stream around solve_sinkhorn, L2
    flushed before each call, as bench.py times it);
  * the wall time of back-to-back calls (host overhead included);
  * the device time of the solve kernel alone (events around a raw
    otk_solve_pointcloud call with prebuilt arguments).
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N  # noqa: E402
from paper_2201_12324_b200 import sinkhorn as S  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(int(os.environ.get("CFG", "1")))
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
prob = otk.LinearProblem(otk.PointCloudGeometry(xd, yd), wl.a, wl.b)
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
for label, kw in (("fixed100", dict(threshold=1e-300, max_iters=100)),
                  ("tolerance", dict(threshold=wl.threshold, max_iters=wl.max_iters))):
    def solve():
        return otk.solve_sinkhorn(prob, wl.eps, **kw)
    for _ in range(20):
        out = solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(50):
        flush.fill_(1.0)
        e0.record()
        solve()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        solve()
    wall = (time.perf_counter() - t0) / 50 * 1e3
    # raw entry, prebuilt args (the native call alone)
    captured = {}
    real = N.lib()

    class Spy:
        def __getattr__(self, name):
            if name == "otk_solve_pointcloud":
                def spy(ptr):
                    captured["args"] = ctypes.cast(ptr, ctypes.POINTER(N.SolveArgs)).contents
                    return real.otk_solve_pointcloud(ptr)
                return spy
            return getattr(real, name)
    saved = S.N.lib
    S.N.lib = lambda: Spy()
    try:
        solve()
    finally:
        S.N.lib = saved
    A = captured["args"]
    t0 = time.perf_counter()
    for _ in range(50):
        real.otk_solve_pointcloud(ctypes.byref(A))
    raw = (time.perf_counter() - t0) / 50 * 1e3
    print(f"{label}: iterations={out.iterations} launches={A.launches} bench-step median "
          f"{np.median(ts):.3f} ms (min {np.min(ts):.3f}); wall {wall:.3f} ms/call; raw native call "
          f"{raw:.3f} ms", flush=True)
