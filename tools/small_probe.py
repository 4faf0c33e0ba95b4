import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2201_12324_b200 as otk
from paper_2201_12324_b200 import workloads
wl = workloads.make(1)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda()))
for _ in range(3): otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=200)
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(10): out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=200)
torch.cuda.synchronize(); print(os.environ.get("OTK_SMALL_PROBE","0"), "%.3f ms per 200-it solve" % ((time.perf_counter()-t0)*100), out.iterations)
