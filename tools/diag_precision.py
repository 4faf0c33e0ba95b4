"""Diagnose float32 vs float64 accuracy of the SIMT / TC paths on a golden solve."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "solve_cfg5_small"
fx = load_golden(name)
wl = getattr(workloads, str(fx["gen"]))(**json.loads(str(fx["kw"])))
thr = float(fx["threshold"]) if "threshold" in fx else 1e-300
mi = int(fx["max_iters"]) if "max_iters" in fx else int(fx["iters"])
geom64 = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
a = oracle.as_weights(wl.a, wl.shape[0])
b = oracle.as_weights(wl.b, wl.shape[1])
for impl in ("simt", "tc"):
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    out = otk.solve_sinkhorn(prob, float(fx["eps"]), threshold=thr, max_iters=mi, impl=impl)
    ef = np.max(np.abs(out.f - fx["f"])) / np.max(np.abs(fx["f"]))
    eg = np.max(np.abs(out.g - fx["g"])) / np.max(np.abs(fx["g"]))
    c = otk.reg_ot_cost(out, prob)
    # cost of OUR potentials evaluated by the float64 oracle
    c64 = oracle.reg_ot_cost(geom64, out.f, out.g, a, b, out.eps)
    print(f"{impl}: iters={out.iterations} f_rel={ef:.2e} g_rel={eg:.2e} "
          f"cost_rel={c.transport_cost / float(fx['transport']) - 1:.2e} "
          f"cost(our f,g; f64 eval)_rel={c64[0] / float(fx['transport']) - 1:.2e} "
          f"dual_rel={c.dual_objective / float(fx['dual']) - 1:.2e}")
    # one half-step at the golden potentials
    geom = otk.PointCloudGeometry(wl.x, wl.y)
    from paper_2201_12324_b200 import _native as N
    geom.impl_flags = N.OTK_IMPL_TC if impl == "tc" else N.OTK_IMPL_SIMT
    r = geom.apply_lse_kernel(np.zeros(wl.shape[0]), fx["g"], float(fx["eps"]), "rows")
    r64 = geom64.apply_lse_kernel(np.zeros(wl.shape[0]), fx["g"], float(fx["eps"]), "rows")
    print(f"   half-step rows at golden g: abs err max {np.max(np.abs(r - r64)):.3e} "
          f"mean {np.mean(r - r64):.3e} (|ref| {np.max(np.abs(r64)):.3f})")
