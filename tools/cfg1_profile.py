"""cfg1 (2048^2, d = 3): where a public-API solve spends its time.

Prints, for the 100-iteration fixed solve and the tolerance solve:
  * the bench step (CUDA events on torch's stream around solve_sinkhorn, L2
    flushed before each call, as bench.py times it);
  * the wall time of back-to-back calls (host overhead included).
The solve kernel's own duration comes from the ncu launch list.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
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
    print(f"{label}: iterations={out.iterations} bench-step median "
          f"{np.median(ts):.3f} ms (min {np.min(ts):.3f}); wall {wall:.3f} ms/call", flush=True)
