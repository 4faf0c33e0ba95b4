"""Accuracy and speed of the tcgen05 kernel's accumulator layouts (OTK_TC_VARIANT).

For d in {64, 128, 256, 1024}: the half-step error vs the float64 oracle (the
cfg-like regimes of tools/diag_tc_bias.py) and, for the golden small solves,
the relative f/g/cost errors.  usage: python tools/diag_variants.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from conftest import load_golden  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402


def half_step_err(d, variant, sphere):
    rng = np.random.default_rng(d)
    n = m = 512
    x = rng.standard_normal((n, d))
    if sphere:
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        y = x + 0.3 * rng.standard_normal((m, d)) / np.sqrt(d)
        y /= np.linalg.norm(y, axis=1, keepdims=True)
        eps = 0.02
    else:
        y = 1.5 * rng.standard_normal((m, d))
        eps = 0.05 * 3.25 * d
    x, y = x.astype(np.float32), y.astype(np.float32)
    ref = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64)).apply_lse_kernel(
        np.zeros(n), np.zeros(m), eps, "rows")
    os.environ["OTK_TC_VARIANT"] = str(variant)
    g = otk.PointCloudGeometry(x, y)
    g.impl_flags = N.OTK_IMPL_TC
    r = g.apply_lse_kernel(np.zeros(n), np.zeros(m), eps, "rows")
    e = r - ref
    return np.mean(e), np.max(np.abs(e)) / np.max(np.abs(ref))


def solve_err(name, variant):
    fx = load_golden(name)
    wl = getattr(workloads, str(fx["gen"]))(**json.loads(str(fx["kw"])))
    thr = float(fx["threshold"]) if "threshold" in fx else 1e-300
    mi = int(fx["max_iters"]) if "max_iters" in fx else int(fx["iters"])
    os.environ["OTK_TC_VARIANT"] = str(variant)
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    out = otk.solve_sinkhorn(prob, float(fx["eps"]), threshold=thr, max_iters=mi, impl="tc")
    ef = np.max(np.abs(out.f - fx["f"])) / np.max(np.abs(fx["f"]))
    eg = np.max(np.abs(out.g - fx["g"])) / np.max(np.abs(fx["g"]))
    c = otk.reg_ot_cost(out, prob)
    return ef, eg, c.transport_cost / float(fx["transport"]) - 1, out.iterations


def main():
    for d in (64, 128, 256, 1024):
        for v in (1, 2, 4):
            if v == 4 and d <= 128:
                continue
            for sphere in (False, True):
                mean, rel = half_step_err(d, v, sphere)
                print(f"d={d:5d} V{v} {'sphere' if sphere else 'gauss '}: mean err {mean:+.2e} "
                      f"max rel {rel:.2e}", flush=True)
    for name in ("solve_cfg2_small", "solve_cfg4_small", "solve_cfg5_small"):
        for v in (1, 2, 4):
            try:
                ef, eg, ec, it = solve_err(name, v)
                print(f"{name} V{v}: f {ef:.2e} g {eg:.2e} cost {ec:+.2e} iters {it}", flush=True)
            except Exception as exc:  # noqa: BLE001
                print(f"{name} V{v}: {exc}", flush=True)


if __name__ == "__main__":
    main()
