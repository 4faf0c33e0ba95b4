"""Medium problems are launch/host-bound: per-iteration wall time of fixed-iteration
solves vs problem size (general tcgen05 loop, d = 64)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

for n in (1024, 2048, 4096, 8192, 16384):
    wl = workloads.cfg2(n=n, m=n, d=64)
    prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(),
                                                    torch.from_numpy(wl.y).cuda()))
    for its in (10, 100):
        for _ in range(2):
            otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=its, fixed_iters=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=its, fixed_iters=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"n=m={n:6d} its={its:4d}: {dt * 1e3:8.3f} ms per solve, {dt / its * 1e6:8.1f} us per iteration",
              flush=True)
