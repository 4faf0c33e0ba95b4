"""Save a GPU tolerance solve's potentials for the float64 converged-flag check.

    python tools/dump_potentials.py 2 4 5      # on the GPU box -> gpurun_out/pot_cfg{k}.npz

Then, in the build container (reference present):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fullsize_golden.py \
        conv:2:gpurun_out/pot_cfg2.npz ...

which evaluates the reference's check pass (sinkhorn.py:181-186) in float64 at
these potentials and writes tests/golden/conv_cfg{k}.npz.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402


def main():
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for k in map(int, sys.argv[1:]):
        wl = workloads.make(k)
        prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
        out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
        path = os.path.join(ROOT, "gpurun_out", f"pot_cfg{k}.npz")
        np.savez_compressed(path, f=out.f.astype(np.float32), g=out.g.astype(np.float32),
                            iterations=np.array(out.iterations), gpu_error=np.array(out.errors[-1]),
                            gpu_dual=np.array(out.dual_trace[-1]),
                            gpu_converged=np.array(out.converged))
        print(f"cfg{k}: iterations={out.iterations} converged={out.converged} "
              f"errors={list(out.errors)} -> {path}", flush=True)


if __name__ == "__main__":
    main()
