"""cfg3 batched solve time vs the persistent kernel's grid (OTK_DENSE_GRID)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.cfg3()
xd, yd = torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda()
for grid in sys.argv[1:]:
    os.environ["OTK_DENSE_GRID"] = grid
    if grid == "lockstep":
        os.environ["OTK_DENSE_LOCKSTEP"] = "1"
    for _ in range(3):
        otk.solve_sinkhorn_batched(xd, yd, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = otk.solve_sinkhorn_batched(xd, yd, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
    e1.record()
    torch.cuda.synchronize()
    print(f"grid {grid}: {e0.elapsed_time(e1) / 5:.2f} ms per solve, max iters {out.iterations.max()}",
          flush=True)
    os.environ.pop("OTK_DENSE_LOCKSTEP", None)
