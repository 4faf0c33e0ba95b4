"""cfg1 solves of several lengths through the public API: the short command behind the ncu capture of
solve_small_kernel.  With a library built by `tools/variant_small.sh abx/count.so -DOTK_SMALL_COUNT_BUILDS`
(OTK_LIB=abx/count.so) OTK_SMALL_DEBUG prints how often CTA 0 rebuilt its stored terms (cfg1: x role 2, y role 1)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2201_12324_b200 as otk
from paper_2201_12324_b200 import workloads
wl = workloads.make(1)
dev = torch.device("cuda", 0)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)))
os.environ["OTK_SMALL_DEBUG"] = "1"
for its in (5, 10, 50, 100, 400):
    otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=its)
