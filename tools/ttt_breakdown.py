"""cfg2 time-to-tolerance: event-timed solves, then one more solve for a launch list
(run under `ncu --metrics gpu__time_duration.sum` to see where the time goes)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(2)
dev = torch.device("cuda", 0)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).to(dev),
                                                torch.from_numpy(wl.y).to(dev)))


def solve():
    return otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)


flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    solve()
times, outs = bench.timed_steps(solve, 5, dev, flush)
print("ttt ms", [round(t * 1e3, 2) for t in times], "iters", outs[-1].iterations, flush=True)
torch.cuda.synchronize()
solve()
torch.cuda.synchronize()
