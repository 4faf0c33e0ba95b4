"""cfg1 (2048^2, d = 3): where a public-API solve spends its time.

Prints, for the 100-iteration fixed solve and the tolerance solve:
  * the bench step (CUDA events on torch's stream around solve_sinkhorn, L2
    flushed before each call, as bench.py times it);
  * the wall time of back-to-back calls (host overhead included).
The solve kernel's own duration comes from the ncu launch list.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(int(os.environ.get("CFG", "1")))
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
prob = otk.LinearProblem(otk.PointCloudGeometry(xd, yd), wl.a, wl.b)
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
t_w = time.perf_counter()  # bring the clocks up before anything is timed
while time.perf_counter() - t_w < 1.5:
    flush.fill_(0.0)
torch.cuda.synchronize()
for label, kw in (("fixed100", dict(threshold=1e-300, max_iters=100)),
                  ("tolerance", dict(threshold=wl.threshold, max_iters=wl.max_iters))):
    def solve():
        return otk.solve_sinkhorn(prob, wl.eps, **kw)
    for _ in range(20):
        out = solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(50):
        flush.fill_(1.0)
        e0.record()
        solve()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        solve()
    wall = (time.perf_counter() - t0) / 50 * 1e3
    print(f"{label}: iterations={out.iterations} bench-step median "
          f"{np.median(ts):.3f} ms (min {np.min(ts):.3f}); wall {wall:.3f} ms/call", flush=True)
# fixed overhead vs per-iteration cost: wall time of back-to-back solves at several iteration counts
pts = []
for its in (10, 50, 100, 200, 400):
    for _ in range(5):
        otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=its)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(40):
        otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=its)
    pts.append((its, (time.perf_counter() - t0) / 40 * 1e6))
slope, icpt = np.polyfit([p[0] for p in pts], [p[1] for p in pts], 1)
print("wall us by iterations:", " ".join(f"{i}:{t:.0f}" for i, t in pts),
      f"-> {slope:.2f} us per iteration + {icpt:.0f} us per call", flush=True)
# where the per-call time goes: the native call alone vs the whole Python entry (10-iteration solves)
from paper_2201_12324_b200 import _native as N  # noqa: E402
lib = N.lib()
real = lib.otk_solve_pointcloud
spent = []


def timed(arg):
    t0 = time.perf_counter()
    rc = real(arg)
    spent.append(time.perf_counter() - t0)
    return rc


lib.otk_solve_pointcloud = timed
try:
    t0 = time.perf_counter()
    for _ in range(200):
        otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=10)
    whole = (time.perf_counter() - t0) / 200 * 1e6
finally:
    lib.otk_solve_pointcloud = real
print(f"10-iteration solve: {whole:.1f} us per call, of which the native call {np.median(spent) * 1e6:.1f} us "
      f"(Python around it {whole - np.median(spent) * 1e6:.1f} us)", flush=True)
