"""Stored-kernel vs plain persistent small solve vs the float64 oracle on one fuzz case, by iteration count."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402


def replay(seed, want):
    rng = np.random.default_rng(seed)
    for c in range(want + 1):
        d = int(rng.choice([2, 3, 5, 16, 33, 64, 100, 128, 200, 300, 520]))
        n = int(rng.integers(1, 900))
        m = int(rng.integers(1, 900))
        off = float(rng.choice([0.0, 0.0, 10.0, 100.0, 1000.0]))
        x = (rng.standard_normal((n, d)) * float(rng.choice([0.3, 1.0, 4.0])) + off).astype(np.float32)
        y = (rng.standard_normal((m, d)) * float(rng.choice([0.5, 1.0, 2.0])) + rng.uniform(-1, 1)
             + off).astype(np.float32)
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


if sys.argv[1] == "long":  # the long-run test problem (tests/test_gpu_parity.py): n m [iteration counts...]
    rng = np.random.default_rng(5)
    n, m, d = int(sys.argv[2]), int(sys.argv[3]), 3
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.5).astype(np.float32)
    a = b = g0 = None
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = 0.5 * float(np.mean(geom64.cost_matrix()))
    counts = [int(v) for v in sys.argv[4:]] or [50, 100, 200, 400, 600]
else:
    x, y, a, b, eps, its, g0 = replay(int(sys.argv[1]), int(sys.argv[2]))
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    counts = [1, 2, 3, 4, 6, 10, its]
sc = eps * np.log(2)
for k in counts:
    ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-300, max_iters=k,
                          g_init=None if g0 is None else g0.astype(np.float64))
    row = []
    for st in ("1", "0"):
        os.environ["OTK_SMALL_STORED"] = st
        geom_ = otk.PointCloudGeometry(x, y)
        if st == "0" and x.shape[1] > 19:  # no plain small solve beyond 19 coordinates: the general loop
            from paper_2201_12324_b200 import _native as N
            geom_.impl_flags = N.OTK_IMPL_NOPERSIST
        prob = otk.LinearProblem(geom_, a, b)
        out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=k, g_init=g0)
        fin = np.isfinite(ref["g"])
        ff = np.isfinite(ref["f"])
        row.append("f mean %+.2e max %.2e | g mean %+.2e max %.2e" % (
            ((out.f - ref["f"])[ff] / sc).mean(), np.abs((out.f - ref["f"])[ff] / sc).max(),
            ((out.g - ref["g"])[fin] / sc).mean(), np.abs((out.g - ref["g"])[fin] / sc).max()))
    print(f"its={k:3d} stored: {row[0]}   plain: {row[1]}   (errors in log2 units)")
