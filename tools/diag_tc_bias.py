"""Measure the systematic error of the TC half-step vs float64 as a function of d."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N  # noqa: E402

for d in (64, 128, 256, 512, 1024):
    rng = np.random.default_rng(d)
    n = m = 512
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = x + 0.3 * rng.standard_normal((m, d)) / np.sqrt(d)   # near pairs: large dots
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    x, y = x.astype(np.float32), y.astype(np.float32)
    eps = 0.02
    ref = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64)).apply_lse_kernel(
        np.zeros(n), np.zeros(m), eps, "rows")
    out = {}
    for impl, fl in (("simt", N.OTK_IMPL_SIMT), ("tc", N.OTK_IMPL_TC)):
        g = otk.PointCloudGeometry(x, y)
        g.impl_flags = fl
        r = g.apply_lse_kernel(np.zeros(n), np.zeros(m), eps, "rows")
        e = r - ref
        out[impl] = f"mean {np.mean(e):+.2e} max {np.max(np.abs(e)):.2e}"
    print(f"d={d:5d}  simt: {out['simt']}   tc: {out['tc']}")
