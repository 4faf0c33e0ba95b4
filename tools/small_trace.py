"""Phase timeline of the persistent small solve (cfg1 shape) from the
OTK_SMALL_TRACE globaltimer stamps: per half-step, the spread of CTA arrival,
exchange wait, cell pass, reduction and publish (medians over CTAs, ns)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402

wl = workloads.make(1)
dev = torch.device("cuda", 0)
prob = otk.LinearProblem(otk.PointCloudGeometry(torch.from_numpy(wl.x).to(dev),
                                                torch.from_numpy(wl.y).to(dev)))
for _ in range(3):
    otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=25)
path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["OTK_SMALL_TRACE"] = path
otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=25)
del os.environ["OTK_SMALL_TRACE"]
G = torch.cuda.get_device_properties(0).multi_processor_count
T = np.fromfile(path, dtype=np.uint64).reshape(64, G, 8).astype(np.int64)
rows = []
slow = []
for s in range(6, 48):
    live = T[s, :, 4] > 0
    if live.sum() < 2 or not (T[s - 1, :, 4] > 0).any():
        continue
    t = T[s, live]
    prev_pub = T[s - 1, T[s - 1, :, 4] > 0, 4].max()
    period = t[:, 4].max() - prev_pub
    wait = np.median(t[:, 1] - t[:, 0])
    cells = np.median(t[:, 2] - t[:, 1])
    red = np.median(t[:, 3] - t[:, 2])
    fin = np.median(t[:, 4] - t[:, 3])
    ent = np.median(t[:, 0] - prev_pub)
    rows.append((s, period, ent, wait, cells, red, fin, t[:, 1].max() - prev_pub))
    k = int(np.argmax(t[:, 4]))  # the CTA that published last: its own phases
    slow.append((s, t[k, 0] - prev_pub, t[k, 1] - t[k, 0], t[k, 2] - t[k, 1], t[k, 3] - t[k, 2],
                 t[k, 4] - t[k, 3], np.median(t[:, 4]) - prev_pub, t[:, 4].min() - prev_pub))
print("step period  entry-after-last-pub  wait  cells  reduce  finalize  last-ready-after-last-pub (ns)")
for r in rows:
    print("%4d %6d %8d %8d %6d %6d %6d %8d" % r)
a = np.array(rows)[:, 1:]
print("median", np.median(a, axis=0).astype(int))
print("last publisher of each step: entry-after-last-pub wait cells reduce finalize | median / first publish after last pub")
for r in slow[-16:]:
    print("%4d %8d %6d %6d %6d %6d | %6d %6d" % r)
print("median", np.median(np.array(slow)[:, 1:], axis=0).astype(int))
print("check steps: finalize->slot words published, ->decision seen (ns, median over CTAs); last CTA decided after the last publish")
for s_ in range(6, 64):
    live = (T[s_, :, 7] > 0) & (T[s_, :, 4] > 0)
    if live.sum() > 1:
        t = T[s_, live]
        print("%4d %6d %6d | %6d" % (s_, np.median(t[:, 5] - t[:, 4]), np.median(t[:, 7] - t[:, 5]),
                                   t[:, 7].max() - t[:, 4].max()))
print("check steps, relative to the last CTA's end of the f(t+1) half-step: CTA 0 words out / gathered / decided; other CTAs decided (median, max)")
for s_ in range(6, 64):
    live = (T[s_, :, 7] > 0) & (T[s_, :, 4] > 0)
    if live.sum() > 1 and T[s_, 0, 6] > 0:
        t4 = T[s_, live, 4].max()
        oth = T[s_, live, 7][1:]
        print("%4d %6d %6d %6d | %6d %6d" % (s_, T[s_, 0, 5] - t4, T[s_, 0, 6] - t4, T[s_, 0, 7] - t4,
                                           np.median(oth) - t4, oth.max() - t4))
