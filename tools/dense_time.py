"""Time the batched dense row half-step (cfg3) -- bench.dense_roofline."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_12324_b200 import _native as N, workloads  # noqa: E402

wl = workloads.cfg3()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
B, n, d = wl.x.shape
m = wl.y.shape[1]
C = torch.empty((B, n, m), dtype=torch.float32, device=dev)
N.check(N.lib().otk_dense_cost(N.ptr(xd), N.ptr(yd), B, n, m, d, 0, N.ptr(C), None,
                               torch.cuda.current_stream().cuda_stream))
r = bench.dense_roofline(C, wl, reps=20)
print(f"{r['kernel']}: {r['kernel_ms'] * 1e3:.1f} us  {r['achieved']:.0f} GB/s  frac {r['frac']:.3f}  "
      f"read-only roof {r['read_only_gbs']:.0f} GB/s -> {r['read_only_frac']:.3f}")
