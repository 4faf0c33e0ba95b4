"""CTA-pair (cta_group::2) tcgen05 kernel vs the 1-CTA kernel: outputs and time.

usage: python tools/pair_check.py   (OTK_TC_PAIR is toggled in-process)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N  # noqa: E402


def half_steps(x, y, f, g, eps):
    geom = otk.PointCloudGeometry(x, y)
    geom.impl_flags = N.OTK_IMPL_TC
    return geom.apply_lse_kernel(f, g, eps, "rows"), geom.apply_lse_kernel(f, g, eps, "cols")


def main():
    rng = np.random.default_rng(0)
    for n, m, d in ((128, 256, 64), (256, 256, 64), (300, 517, 40), (1000, 700, 128),
                    (129, 1031, 96), (4096, 4096, 64), (5000, 3000, 100)):
        x = rng.standard_normal((n, d)).astype(np.float32)
        y = (1.3 * rng.standard_normal((m, d)) + 0.2).astype(np.float32)
        eps = 0.05 * 3.0 * d
        f = (rng.standard_normal(n) * eps).astype(np.float32).astype(np.float64)
        g = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
        os.environ["OTK_TC_PAIR"] = "0"
        r0, c0 = half_steps(x, y, f, g, eps)
        os.environ["OTK_TC_PAIR"] = "1"
        r1, c1 = half_steps(x, y, f, g, eps)
        torch.cuda.synchronize()
        dr = np.max(np.abs(r1 - r0)) / np.max(np.abs(r0))
        dc = np.max(np.abs(c1 - c0)) / np.max(np.abs(c0))
        print(f"n={n} m={m} d={d}: rows rel diff {dr:.2e} cols {dc:.2e} "
              f"bitwise {np.array_equal(r0, r1) and np.array_equal(c0, c1)}", flush=True)


if __name__ == "__main__":
    main()
