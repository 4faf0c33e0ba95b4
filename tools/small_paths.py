"""cfg1-size solve: persistent one-kernel solve vs the general loop (TC / FP32 kernels)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402

for n in (2048, 4096, 8192):
    wl = workloads.cfg1(n=n, m=n)
    xd, yd = torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda()
    for label, flags in (("persistent", 0), ("loop+tc", N.OTK_IMPL_NOPERSIST | N.OTK_IMPL_TC),
                         ("loop+fp32", N.OTK_IMPL_NOPERSIST | N.OTK_IMPL_SIMT)):
        geom = otk.PointCloudGeometry(xd, yd)
        geom.impl_flags = flags
        prob = otk.LinearProblem(geom)
        for _ in range(3):
            otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
        torch.cuda.synchronize()
        print(f"n={n} {label:10s} {1e3 * (time.perf_counter() - t0) / 10:.3f} ms  iters {out.iterations}",
              flush=True)
