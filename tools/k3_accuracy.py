"""Batched solvers vs the float64 oracle: K3c scaling domain (default), K3c log domain, K3p."""
import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import oracle
import paper_2201_12324_b200 as otk
for (n, m) in ((130, 68), (512, 512), (700, 300)):
    rng = np.random.default_rng(n + m)
    B, d = 20, 5
    x = rng.standard_normal((B, n, d)).astype(np.float32)
    y = (rng.standard_normal((B, m, d)) + rng.uniform(-1, 1, (B, 1, d))).astype(np.float32)
    eps = np.array([0.05 * np.mean(np.sum((x[k, :64, None] - y[k, None, :64]) ** 2, -1)) for k in range(B)])
    res = {}
    for label, env in (("scaled", {"OTK_DENSE_KERNEL": "cluster"}), ("log", {"OTK_DENSE_KERNEL": "cluster", "OTK_DENSE_DOMAIN": "log"}), ("cta", {"OTK_DENSE_KERNEL": "cta"})):
        for k in ("OTK_DENSE_KERNEL", "OTK_DENSE_DOMAIN"):
            os.environ.pop(k, None)
        os.environ.update(env)
        res[label] = otk.solve_sinkhorn_batched(x, y, eps, threshold=1e-300, max_iters=37)
    worst = {k: 0.0 for k in res}
    for b in range(B):
        C = ((x[b].astype(np.float64)[:, None, :] - y[b].astype(np.float64)[None]) ** 2).sum(-1)
        ref = oracle.sinkhorn(oracle.DenseOracle(C), None, None, float(eps[b]), threshold=1e-300, max_iters=37)
        for k, o in res.items():
            e = max(np.max(np.abs(o.f[b] - ref["f"])) / np.max(np.abs(ref["f"])), np.max(np.abs(o.g[b] - ref["g"])) / np.max(np.abs(ref["g"])))
            worst[k] = max(worst[k], e)
    print(n, m, {k: f"{v:.2e}" for k, v in worst.items()}, flush=True)
