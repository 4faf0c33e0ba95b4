"""Per-iteration cost of the persistent small solve (cfg1 shape): time fixed
100- and 300-iteration solves with CUDA events and report the difference / 200
(launch + setup cancel).  Env knob read by the library: OTK_SMALL_PROBE=1 (timing
probe: skip the passes over the cells, see solve_small.cu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = workloads.make(cfg)
dev = torch.device("cuda", 0)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).to(dev),
                                                torch.from_numpy(wl.y).to(dev)))


def t_solve(iters, reps=10):
    for _ in range(3):
        otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=iters)
    best = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=iters)
        e.record()
        torch.cuda.synchronize()
        best.append(s.elapsed_time(e))
    best.sort()
    return best[len(best) // 2], out.iterations


t1, i1 = t_solve(100)
t3, i3 = t_solve(300)
tag = "PROBE=%s" % os.environ.get("OTK_SMALL_PROBE", "0")
print("%s  100-it %.3f ms  300-it %.3f ms  per-iteration %.2f us (iters %d/%d)"
      % (tag, t1, t3, (t3 - t1) / (i3 - i1) * 1e3, i1, i3), flush=True)
