"""Launch the dominant kernel (one rows half-step, otk_lse_partial) of a config
a few times -- a short command for `ncu --set full -k regex:lse_` captures.

usage: python tools/prof_half_step.py [--config 2] [--reps 5] [--kernel auto|simt|tc]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tc", "tc-noanchor"])
    ap.add_argument("--n", type=int)
    ap.add_argument("--m", type=int)
    ap.add_argument("--d", type=int)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    kw = {k: getattr(args, k) for k in ("n", "m", "d") if getattr(args, k) is not None}
    wl = workloads.make(args.config, **kw)
    geom = otk.PointCloudGeometry(torch.from_numpy(wl.x).cuda(), torch.from_numpy(wl.y).cuda())
    if args.kernel == "simt":
        geom.impl_flags = N.OTK_IMPL_SIMT
    elif args.kernel == "tc":
        geom.impl_flags = N.OTK_IMPL_TC
    elif args.kernel == "tc-noanchor":
        geom.impl_flags = N.OTK_IMPL_TC | N.OTK_IMPL_NOANCHOR
    r = bench.online_roofline(geom, wl, reps=args.reps)
    print(f"config {args.config}: {r['kernel_ms']:.3f} ms per half-step, "
          f"{r['pipes']['cells_per_s']:.3e} cells/s, {r['bound']} frac {r['frac']:.3f}")


if __name__ == "__main__":
    main()
