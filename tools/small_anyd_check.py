"""Any-d small solve vs the tcgen05 loop (OTK_IMPL_NOPERSIST): 30 fixed iterations, time and agreement."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2201_12324_b200 as otk
from paper_2201_12324_b200 import workloads, _native as N
for d, n, m in ((512, 2048, 2048), (256, 2048, 1500), (20, 2048, 2048), (511, 1000, 2048), (130, 2048, 2048),
                (67, 1500, 1333)):
    wl = workloads.cfg2(n=n, m=m, d=d)
    xd, yd = torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda()
    res = {}
    for name, fl in (("small", 0), ("tcloop", N.OTK_IMPL_NOPERSIST)):
        g = otk.PointCloudGeometry(xd, yd); g.impl_flags = fl
        prob = otk.LinearProblem(g)
        out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=30, fixed_iters=True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(5):
            out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=30, fixed_iters=True)
        torch.cuda.synchronize()
        res[name] = (out, (time.perf_counter() - t0) / 5 * 1e3)
    a, b = res["small"][0], res["tcloop"][0]
    rel = lambda u, v: np.max(np.abs(u - v)) / np.max(np.abs(v))
    print(f"d={d} n={n} m={m}: small {res['small'][1]:.3f} ms, tc loop {res['tcloop'][1]:.3f} ms per 30 iterations; "
          f"f diff {rel(a.f, b.f):.1e} g diff {rel(a.g, b.g):.1e}", flush=True)
