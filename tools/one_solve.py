"""Run K warm solves then one timed solve of a config (for ncu launch lists)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workloads.make(cfg)
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
prob = otk.LinearProblem(otk.PointCloudGeometry(xd, yd), wl.a, wl.b)
for _ in range(3):
    otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
e1.record()
torch.cuda.synchronize()
print(f"solve: events {e0.elapsed_time(e1):.2f} ms, wall {1e3 * (time.perf_counter() - t0):.2f} ms, "
      f"iterations {out.iterations}")
