"""Re-run one case of tools/fuzz_parity.py with diagnostics (which stage carries the error)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N  # noqa: E402


def replay(seed, want):
    rng = np.random.default_rng(seed)
    for c in range(want + 1):
        d = int(rng.choice([2, 3, 5, 16, 33, 64, 100, 128, 200, 300, 520]))
        n = int(rng.integers(1, 900))
        m = int(rng.integers(1, 900))
        x = rng.standard_normal((n, d)).astype(np.float32) * float(rng.choice([0.3, 1.0, 4.0]))
        y = (rng.standard_normal((m, d)) * float(rng.choice([0.5, 1.0, 2.0])) + rng.uniform(-1, 1)).astype(np.float32)
        a = rng.uniform(0.5, 1.5, n)
        b = rng.uniform(0.5, 1.5, m)
        if rng.random() < 0.4 and n > 2:
            a[rng.choice(n, max(1, n // 10), replace=False)] = 0.0
        if rng.random() < 0.4 and m > 2:
            b[rng.choice(m, max(1, m // 10), replace=False)] = 0.0
        a /= a.sum()
        b /= b.sum()
        k = min(n, m, 64)
        mc = float(np.mean(np.sum((x[:k, None, :] - y[None, :k, :]) ** 2, axis=-1)))
        eps = float(rng.choice([0.01, 0.05, 0.5])) * max(mc, 1e-3)
        its = int(rng.integers(3, 40))
        g0 = None
        if rng.random() < 0.3:
            g0 = (rng.standard_normal(m) * eps * float(rng.choice([1.0, 50.0]))).astype(np.float32)
    return x, y, a, b, eps, its, g0


def main(seed, case):
    x, y, a, b, eps, its, g0 = replay(seed, case)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-300, max_iters=its,
                          g_init=None if g0 is None else g0.astype(np.float64))
    ref_cost = oracle.reg_ot_cost(geom64, ref["f"], ref["g"], a, b, eps)
    print("n m d", x.shape[0], y.shape[0], x.shape[1], "eps", eps, "its", its, "ref cost", ref_cost)
    for impl in ("auto", "simt", "tc"):
        prob = otk.LinearProblem(otk.PointCloudGeometry(x, y), a, b)
        out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=its, g_init=g0, impl=impl)
        cost = otk.reg_ot_cost(out, prob)
        # the oracle's cost formula on OUR potentials: separates potential error from cost-kernel error
        oc = oracle.reg_ot_cost(geom64, out.f, out.g, a, b, eps)
        fin = np.isfinite(ref["f"])
        print(f"{impl:5s} f {np.max(np.abs(out.f[fin]-ref['f'][fin]))/np.max(np.abs(ref['f'][fin])):.2e} "
              f"transport {cost.transport_cost / ref_cost[0] - 1:+.2e} "
              f"(oracle formula on our f,g: {oc[0] / ref_cost[0] - 1:+.2e}) dual {cost.dual_objective / ref_cost[1] - 1:+.2e}")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
