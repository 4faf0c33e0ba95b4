"""One cfg3 batched solve (for ncu -k regex:dense_cluster)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.cfg3()
for _ in range(2):
    otk.solve_sinkhorn_batched(wl.x, wl.y, wl.eps, threshold=1e-3, max_iters=500)
