import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2201_12324_b200 as otk
from paper_2201_12324_b200 import workloads
wl = workloads.make(2)
xh = torch.from_numpy(wl.x).pin_memory(); yh = torch.from_numpy(wl.y).pin_memory()
def step():
    t0=time.perf_counter()
    geom = otk.PointCloudGeometry(xh, yh); torch.cuda.synchronize(); t1=time.perf_counter()
    prob = otk.LinearProblem(geom, wl.a, wl.b); geom._clouds(); prob._weights(); torch.cuda.synchronize(); t2=time.perf_counter()
    out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters); t3=time.perf_counter()
    return (t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3
for _ in range(3): step()
for _ in range(3): print(["%.2f"%v for v in step()])
