"""Same-box A/B of the one-launch batched solve (cfg3) across library builds.

    python tools/ab_dense.py lib1.so [lib2.so ...]

Loads each build with ctypes directly (older builds may lack newer symbols),
runs otk_solve_dense_batched on the full cfg3 batch (fixed 30 iterations and
the tolerance run) and prints the median time of 10 launches (CUDA events)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_12324_b200 import workloads  # noqa: E402

P, I64, I32, F64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double


def bind(path):
    lib = C.CDLL(path)
    lib.otk_dense_cost.argtypes = [P, P, I64, I64, I64, I32, I32, P, P, P]
    lib.otk_solve_dense_batched.argtypes = [P, I64, I64, I64, P, P, P, P, P, P, P, F64, I32, I32, I32,
                                            P, P, P, P, P, I32, P]
    return lib


wl = workloads.cfg3()
dev = torch.device("cuda", 0)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
B, n, d = wl.x.shape
m = wl.y.shape[1]
st = torch.cuda.current_stream().cuda_stream
a = torch.full((B, n), 1.0 / n, device=dev)
b = torch.full((B, m), 1.0 / m, device=dev)
la, lb = torch.full_like(a, -float(np.log(n))), torch.full_like(b, -float(np.log(m)))
e32 = torch.as_tensor(wl.eps.astype(np.float32), device=dev)
e64 = torch.as_tensor(wl.eps, device=dev)
results = {}
for path in sys.argv[1:]:
    lib = bind(path)
    Cm = torch.empty((B, n, m), device=dev)
    assert lib.otk_dense_cost(xd.data_ptr(), yd.data_ptr(), B, n, m, d, 0, Cm.data_ptr(), None, st) == 0
    for label, thr, mi in (("fixed30", 1e-300, 30), ("tol", wl.threshold, wl.max_iters)):
        mc = mi // 10 + 2
        f, g = torch.empty((B, n), device=dev), torch.empty((B, m), device=dev)
        errs = torch.empty((B, mc), dtype=torch.float64, device=dev)
        duals = torch.empty_like(errs)
        state = torch.zeros((B, 5), dtype=torch.int32, device=dev)

        def launch():
            rc = lib.otk_solve_dense_batched(Cm.data_ptr(), B, n, m, a.data_ptr(), b.data_ptr(),
                                             la.data_ptr(), lb.data_ptr(), e32.data_ptr(), e64.data_ptr(),
                                             None, thr, mi, 10, mc, f.data_ptr(), g.data_ptr(),
                                             errs.data_ptr(), duals.data_ptr(), state.data_ptr(), 0, st)
            assert rc == 0
        for _ in range(3):
            launch()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        its = state[:, 1].cpu().numpy()
        results[(path, label)] = (f.cpu().numpy(), g.cpu().numpy(), its)
        print(f"{os.path.basename(path)} {label}: median {np.median(ts):.3f} ms (min {np.min(ts):.3f}), "
              f"iterations {np.unique(its, return_counts=True)}", flush=True)
if len(sys.argv) > 2:
    p0 = sys.argv[1]
    for p1 in sys.argv[2:]:
        for label in ("fixed30", "tol"):
            f0, g0, i0 = results[(p0, label)]
            f1, g1, i1 = results[(p1, label)]
            df = np.max(np.abs(f1 - f0) / np.max(np.abs(f0), axis=1, keepdims=True))
            print(f"{os.path.basename(p1)} vs {os.path.basename(p0)} {label}: max rel f diff {df:.2e}, "
                  f"same iterations {np.array_equal(i0, i1)}")
