"""cfg1 tolerance solve timed like bench.py (L2 flushed before each, CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(1)
dev = torch.device("cuda", 0)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)))
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
for kw in (dict(threshold=1e-3, max_iters=2000), dict(threshold=1e-300, max_iters=100)):
    solve = lambda: otk.solve_sinkhorn(prob, wl.eps, **kw)  # noqa: E731
    for _ in range(5):
        solve()
    ts, _ = bench.timed_steps(solve, 8, dev, flush)
    print(kw, " ".join(f"{t * 1e3:.3f}" for t in ts), flush=True)
