import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2201_12324_b200 as otk
from paper_2201_12324_b200 import workloads
wl = workloads.make(1)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda()))
for kw in (dict(threshold=1e-3, max_iters=2000), dict(threshold=1e-3, max_iters=40), dict(threshold=1e-300, max_iters=40), dict(threshold=1e-3, max_iters=200)):
    for _ in range(5): out = otk.solve_sinkhorn(prob, wl.eps, **kw)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): out = otk.solve_sinkhorn(prob, wl.eps, **kw)
    torch.cuda.synchronize()
    print(kw, "%.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3), out.iterations, flush=True)
