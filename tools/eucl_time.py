"""sqeucl vs eucl solve time at a cfg2-like shape (fixed iterations), same process.

usage: python tools/eucl_time.py [n] [d] [iters]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    rng = np.random.default_rng(2)
    x = torch.as_tensor(rng.standard_normal((n, d)).astype(np.float32), device="cuda")
    y = torch.as_tensor((1.5 * rng.standard_normal((n, d))).astype(np.float32), device="cuda")
    for cost_fn in ("sqeucl", "eucl", "sqeucl", "eucl"):
        geom = otk.PointCloudGeometry(x, y, cost_fn)
        eps = 0.05 * geom.mean_cost()
        prob = otk.LinearProblem(geom)
        otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=iters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{cost_fn:7s} n={n} d={d}: {dt * 1e3:.1f} ms / {iters} its -> "
              f"{n * n * iters / dt:.3e} cell-updates/s  ({dt / (2 * iters + 1) * 1e3:.2f} ms/half-step)",
              flush=True)


if __name__ == "__main__":
    main()
