"""cfg1: a few persistent one-kernel solves (for ncu -k regex:solve_small)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(1)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(),
                                                torch.from_numpy(wl.y).cuda()))
for _ in range(3):
    out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=200)
torch.cuda.synchronize()
print("iters", out.iterations)
