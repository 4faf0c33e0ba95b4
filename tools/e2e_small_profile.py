"""Host-side cost of one public-API cfg1 solve from pinned host buffers
(the bench e2e step): wall time per call, the device solve time, and a
cProfile of the Python host path."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(1)
xh = torch.from_numpy(wl.x).pin_memory()
yh = torch.from_numpy(wl.y).pin_memory()


def step():
    prob = otk.LinearProblem(otk.PointCloudGeometry(xh, yh), wl.a, wl.b)
    return otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=100)


for _ in range(20):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    step()
torch.cuda.synchronize()
print("public API step: %.3f ms" % ((time.perf_counter() - t0) / 50 * 1e3))
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
