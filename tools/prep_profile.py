"""cfg1: where the public-API time before the solve goes (geometry construction from pinned host
arrays, centring, the eps estimate), wall-clock per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(int(os.environ.get("CFG", "1")))
xh, yh = torch.from_numpy(wl.x).pin_memory(), torch.from_numpy(wl.y).pin_memory()
xd, yd = xh.cuda(), yh.cuda()


def timeit(fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print("geometry from pinned host arrays: %.0f us" % timeit(lambda: otk.PointCloudGeometry(xh, yh)))
print("geometry from device tensors:     %.0f us" % timeit(lambda: otk.PointCloudGeometry(xd, yd)))
print("  + centred points (_points):     %.0f us" % timeit(lambda: otk.PointCloudGeometry(xd, yd)._points()))
print("  + eps estimate (epsilon_default): %.0f us" % timeit(lambda: otk.PointCloudGeometry(xd, yd).epsilon_default))
g = otk.PointCloudGeometry(xd, yd)
prob = otk.LinearProblem(g)
print("LinearProblem + weights:          %.0f us" % timeit(lambda: otk.LinearProblem(otk.PointCloudGeometry(xd, yd))._weights()))
print("tolerance solve on a prepared problem: %.0f us" % timeit(
    lambda: otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)))
