"""Per-iteration wall time of small single problems by d (the persistent
one-kernel solve serves d <= 7; larger d runs the launch-per-half-step loop)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402

rng = np.random.default_rng(0)
for n in (512, 2048):
    for d in (3, 7, 8, 16, 64):
        x = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
        y = torch.from_numpy((rng.standard_normal((n, d)) + 0.3).astype(np.float32)).cuda()
        prob = otk.LinearProblem(otk.PointCloudGeometry(x, y))
        eps = 0.05 * 2 * d
        res = []
        for its in (100, 300):
            for _ in range(2):
                otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=its, inner_iters=its)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=its, inner_iters=its)
            torch.cuda.synchronize()
            res.append((time.perf_counter() - t0) / 5)
        print(f"n=m={n:5d} d={d:3d}: {(res[1] - res[0]) / 200 * 1e6:7.2f} us per iteration", flush=True)
