"""cfg5 (d = 1024): accuracy and speed of the V2 (double-buffered) vs V4
(single-buffered, 3 hi*hi slices) tcgen05 accumulator layouts against the
reference fixtures (tests/golden).  usage: python tools/cfg5_variants.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def main():
    for v in (4, 2):
        os.environ["OTK_TC_VARIANT"] = str(v)
        for name in ("fixed_cfg5_fixed30", "solve_cfg5_small"):
            fx = load_golden(name)
            wl = workloads.cfg5(**json.loads(str(fx["kw"])))
            prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y))
            thr = float(fx["threshold"]) if "threshold" in fx else 1e-300
            mi = int(fx["max_iters"]) if "max_iters" in fx else int(fx["iters"])
            out = otk.solve_sinkhorn(prob, float(fx["eps"]), threshold=thr, max_iters=mi, impl="tc")
            c = otk.reg_ot_cost(out, prob)
            print(f"V{v} {name}: f {rel(out.f, fx['f']):.2e} g {rel(out.g, fx['g']):.2e} "
                  f"transport {abs(c.transport_cost / float(fx['transport']) - 1):.2e} "
                  f"dual {abs(c.dual_objective / float(fx['dual']) - 1):.2e} it {out.iterations}",
                  flush=True)
        fx = load_golden("spot_cfg5")
        wl = workloads.make(5)
        geom = otk.PointCloudGeometry(wl.x, wl.y)
        geom.impl_flags = N.OTK_IMPL_TC
        eps = float(fx["eps"])
        n, m = wl.shape
        r0 = geom.apply_lse_kernel(np.zeros(n), np.zeros(m), eps, "rows")[fx["rows"]]
        rg = geom.apply_lse_kernel(np.zeros(n), fx["g"].astype(np.float64), eps, "rows")[fx["rows"]]
        cf = geom.apply_lse_kernel(fx["f"].astype(np.float64), np.zeros(m), eps, "cols")[fx["cols"]]
        print(f"V{v} spot_cfg5: rows_g0 {rel(r0, fx['rows_g0']):.2e} rows_g {rel(rg, fx['rows_g']):.2e} "
              f"cols_f {rel(cf, fx['cols_f']):.2e}", flush=True)
        geom2 = otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda())
        geom2.impl_flags = N.OTK_IMPL_TC
        r = bench.online_roofline(geom2, wl, reps=5)
        print(f"V{v} cfg5 half-step {r['kernel_ms']:.3f} ms frac {r['frac']:.3f}", flush=True)


if __name__ == "__main__":
    main()
