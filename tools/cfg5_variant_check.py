"""cfg5 at full size: the tcgen05 accumulator layouts (OTK_TC_VARIANT 2 vs the
default 4) against the reference's full-size fixtures (fixed 2 iterations and
the tolerance solve): potentials, transport cost, dual, and half-step time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.cfg5()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
for name in ("full_cfg5_it2", "full_cfg5_tol"):
    fx = load_golden(name)
    prob = otk.LinearProblem(otk.PointCloudGeometry(xd, yd))
    kw = dict(threshold=float(fx.get("threshold", 1e-300)), max_iters=int(fx["max_iters"]))
    for _ in range(2):
        out = otk.solve_sinkhorn(prob, wl.eps, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = otk.solve_sinkhorn(prob, wl.eps, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    c = otk.reg_ot_cost(out, prob)
    ef = np.max(np.abs(out.f - fx["f"])) / np.max(np.abs(fx["f"]))
    eg = np.max(np.abs(out.g - fx["g"])) / np.max(np.abs(fx["g"]))
    print(f"variant={os.environ.get('OTK_TC_VARIANT', 'default')} {name}: iters={out.iterations} "
          f"f {ef:.2e} g {eg:.2e} transport {abs(c.transport_cost / float(fx['transport']) - 1):.2e} "
          f"dual {abs(c.dual_objective / float(fx['dual']) - 1):.2e} solve {dt * 1e3:.1f} ms", flush=True)
