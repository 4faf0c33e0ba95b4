"""Phase timeline of the cluster-resident batched solve (K3c, cfg3) from the
OTK_DENSE_TRACE globaltimer stamps of cluster 0's first problem (rank-0 CTA):
per iteration, rows pass, column partials, cluster barrier, combine, check (ns).
Needs a trace build: tools/build_variant.sh abx/trace.so -DOTK_DENSE_TRACE_BUILD,
then OTK_LIB=abx/trace.so python tools/dense_trace.py."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.cfg3()
for _ in range(2):
    otk.solve_sinkhorn_batched(wl.x, wl.y, wl.eps, threshold=1e-300, max_iters=30)
path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["OTK_DENSE_TRACE"] = path
otk.solve_sinkhorn_batched(wl.x, wl.y, wl.eps, threshold=1e-300, max_iters=30)
T = np.fromfile(path, dtype=np.uint64).reshape(64, 8).astype(np.int64)
print("iter  total  rows  cols  csync  combine  check  (rows: v/drift part)")
for t in range(2, 30):
    if T[t + 1, 0] == 0:
        break
    tot = T[t + 1, 0] - T[t, 0]
    chk = (T[t, 5] - T[t, 4]) if T[t, 5] else 0
    vpart = (T[t, 6] - T[t, 0]) if T[t, 6] else 0
    print("%4d %6d %5d %5d %6d %7d %6d %6d" % (t, tot, T[t, 1] - T[t, 0], T[t, 2] - T[t, 1],
                                               T[t, 3] - T[t, 2], T[t, 4] - T[t, 3], chk, vpart))
print("scaled domain: kernel-slice rebuilds %d, exact column fallbacks %d (whole batch, 30 iterations)"
      % (T[63, 0], T[63, 1]))
