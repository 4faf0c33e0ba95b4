"""Where does a cfg2 solve's time go?  Device-timed solve under variations.

usage: python tools/solve_timing.py [--config 2]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2201_12324_b200 as otk  # noqa: E402
from paper_2201_12324_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    wl = workloads.make(args.config)
    dev = torch.device("cuda", 0)
    xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    if wl.materialised:
        def solve():
            return otk.solve_sinkhorn_batched(xd, yd, wl.eps, threshold=wl.threshold,
                                              max_iters=wl.max_iters)
    else:
        prob = otk.LinearProblem(otk.PointCloudGeometry(xd, yd), wl.a, wl.b)

        def solve():
            return otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold,
                                      max_iters=wl.max_iters)

    for _ in range(3):
        solve()
    for label, fl, clk in (("plain", False, False), ("flush", True, False),
                           ("flush+clock", True, True), ("plain", False, False)):
        sampler = bench.ClockSampler(0) if clk else None
        if sampler:
            sampler.__enter__()
        t_wall = time.perf_counter()
        times, outs = bench.timed_steps(solve, 3, dev, flush) if fl else bench.timed_steps(
            solve, 3, dev, torch.empty(1, device=dev))
        t_wall = time.perf_counter() - t_wall
        if sampler:
            sampler.__exit__()
        print(f"{label:12s} ms/step {[round(t * 1e3, 2) for t in times]} wall/step "
              f"{t_wall / 3 * 1e3:.2f}", flush=True)
    # host-side breakdown of one solve
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = solve()
    t1 = time.perf_counter()
    print(f"one solve wall {1e3 * (t1 - t0):.2f} ms")
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        solve()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
