"""cfg3 public-API batched solve to tolerance from device and from pinned host
inputs (CUDA events around each call, L2 flushed before each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.cfg3()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
xh, yh = torch.from_numpy(wl.x).pin_memory(), torch.from_numpy(wl.y).pin_memory()
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
for name, (x, y), kw in (("device tol", (xd, yd), dict(threshold=1e-3, max_iters=500)),
                         ("pinned tol", (xh, yh), dict(threshold=1e-3, max_iters=500)),
                         ("device 100", (xd, yd), dict(threshold=1e-300, max_iters=100)),
                         ("pinned 100", (xh, yh), dict(threshold=1e-300, max_iters=100))):
    ts = []
    for r in range(6):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = otk.solve_sinkhorn_batched(x, y, wl.eps, **kw)
        _ = out.f
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name}: " + " ".join(f"{t:.2f}" for t in ts[1:]) + f" ms  (iters max {int(out.iterations.max())})",
          flush=True)
