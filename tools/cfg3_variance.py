"""cfg3 (512 x 512^2 batched) step-time spread: the one-launch batched solve
timed step by step, with and without the L2 flush before each step, plus the
cluster plan (K3c cluster size and SMs used)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402

wl = workloads.cfg3()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
c, u = ctypes.c_int32(), ctypes.c_int32()
N.lib().otk_dense_cluster_plan(512, 512, 512, ctypes.byref(c), ctypes.byref(u))
print(f"cluster plan: CL={c.value}, SMs={u.value}", flush=True)
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
for iters in (100, 20):
    for fl in (True, False):
        ts = []
        for k in range(12):
            if fl:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = otk.solve_sinkhorn_batched(xd, yd, wl.eps, threshold=1e-300, max_iters=iters)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"iters={iters} flush={fl}: " + " ".join(f"{t:.2f}" for t in ts), flush=True)
