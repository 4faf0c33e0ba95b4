"""cfg3 step breakdown: cost build (otk_dense_cost) vs the one-launch batched
solve (K3p) vs the whole public-API step, CUDA events, L2 flushed before each."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402
from paper_2201_12324_b200._device import stream  # noqa: E402


def timeit(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


wl = workloads.cfg3()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
B, n, d = wl.x.shape
m = wl.y.shape[1]
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
C = torch.empty((B, n, m), dtype=torch.float32, device=dev)


def cost():
    N.check(N.lib().otk_dense_cost(N.ptr(xd), N.ptr(yd), B, n, m, d, 0, N.ptr(C), None, stream()))


def solve():
    return otk.solve_sinkhorn_batched(xd, yd, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)


for _ in range(3):
    cost()
    solve()
print("dense_cost ms", [round(t, 3) for t in timeit(cost, 5, flush)])
print("full step ms", [round(t, 3) for t in timeit(solve, 5, flush)])
r = bench.dense_roofline(C, wl, reps=5)
print(f"K3p alone {r['kernel_ms']:.3f} ms  {r['achieved']:.0f} GB/s frac {r['frac']:.3f}")
