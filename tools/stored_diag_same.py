"""Same-points small problem (tests/test_gpu_parity.py d=3 same=True): gauge error of stored vs plain by iteration count."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402

d = 3
rng = np.random.default_rng(100 + d)
n = 700
x = rng.standard_normal((n, d)).astype(np.float32)
geom64 = oracle.PointCloudOracle(x.astype(np.float64), x.astype(np.float64))
eps = 0.05 * float(np.mean(geom64.cost_matrix()))
sc = eps * np.log(2)
for k in (1, 2, 3, 5, 10, 20, 30):
    ref = oracle.sinkhorn(geom64, None, None, eps, threshold=1e-300, max_iters=k)
    row = []
    for st in ("1", "0"):
        os.environ["OTK_SMALL_STORED"] = st
        out = otk.solve_sinkhorn(otk.LinearProblem(otk.PointCloudGeometry(x, x)), eps, threshold=1e-300, max_iters=k)
        row.append("f mean %+.2e max %.2e | g mean %+.2e max %.2e" % (
            ((out.f - ref["f"]) / sc).mean(), np.abs((out.f - ref["f"]) / sc).max(),
            ((out.g - ref["g"]) / sc).mean(), np.abs((out.g - ref["g"]) / sc).max()))
    print(f"its={k:3d} stored: {row[0]}   plain: {row[1]}   (log2 units; |f|max {np.abs(ref['f']).max()/sc:.1f} |g|max {np.abs(ref['g']).max()/sc:.1f})")
