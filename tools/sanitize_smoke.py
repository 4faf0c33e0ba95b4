"""Tiny run of every device path, for `compute-sanitizer --tool memcheck|racecheck`.

usage: compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    for d, flags, n, m in ((3, 0, 300, 257),                      # persistent small solve
                           (3, N.OTK_IMPL_NOPERSIST, 300, 257),   # general loop, FP32 kernel
                           (64, 0, 384, 320),                     # tcgen05 V1
                           (200, 0, 256, 200),                    # tcgen05 V2
                           (320, 0, 200, 136)):                   # tcgen05 V4
        x = rng.standard_normal((n, d)).astype(np.float32)
        y = (rng.standard_normal((m, d)) + 0.3).astype(np.float32)
        geom = otk.PointCloudGeometry(x, y)
        geom.impl_flags = flags
        prob = otk.LinearProblem(geom)
        eps = 0.05 * 2.1 * d
        out = otk.solve_sinkhorn(prob, eps, threshold=1e-3, max_iters=30)
        cost = otk.reg_ot_cost(out, prob)
        print(f"d={d} flags={flags:#x}: iters {out.iterations} cost {cost.transport_cost:.5f}",
              flush=True)
    # same points, transport matrix, apply_lse_kernel both axes
    x = rng.standard_normal((200, 3)).astype(np.float32)
    geom = otk.PointCloudGeometry(x, x)
    out = otk.solve_sinkhorn(otk.LinearProblem(geom), 0.3, max_iters=20)
    otk.transport_matrix(out, otk.LinearProblem(geom))
    geom.apply_lse_kernel(np.zeros(200), np.zeros(200), 0.3, "cols")
    # batched dense
    xs = rng.standard_normal((4, 96, 16)).astype(np.float32)
    ys = rng.standard_normal((4, 80, 16)).astype(np.float32)
    outs, costs = otk.solve_sinkhorn_batched(xs, ys, 1.6, threshold=1e-3, max_iters=50,
                                             return_cost=True)
    print("batched iterations", list(outs.iterations), flush=True)
    # dense geometry
    C = rng.uniform(0, 1, (50, 40))
    out = otk.solve_sinkhorn(otk.LinearProblem(otk.DenseGeometry(C)), 0.1, max_iters=40)
    print("dense iterations", out.iterations)
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
