"""Benchmark: Sinkhorn cell-updates/s (n*m*iters/s) and time-to-tolerance.

Default workload = BASELINE.json configs[1] (cfg2: n = m = 65536, d = 64,
fp32, eps = 0.05 x subsample mean, tolerance 1e-3, checks every 10).
One STEP = one complete ``solve_sinkhorn`` to tolerance on inputs already
resident in HBM (so ms_per_step is the time-to-tolerance and
value = n*m*iterations / step time).  Between timed steps L2 is flushed by
writing a 512 MiB buffer (inputs are ~64 MiB, below the 126 MB L2).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config k]

Multi-GPU (torchrun, one rank per GPU): each rank runs an independent
replica of the workload (replicas; the row-sharded NCCL solver is reported
separately) -- value is the sum over ranks of n*m*iters / max-over-ranks time.

``--impl reference`` times the CPU oracle (the numpy restatement of the
reference, oracle/) on a bounded sample of the same workload on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "roofline_traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.05):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm
def cpu_sample_rate(wl, budget_s=12.0, rows=None):
    """Time the oracle (reference restatement) on a bounded sample of one full
    iteration: a rows half-step on `rows` rows and a cols half-step on `rows`
    columns, each reducing over the FULL other axis.  Returns cell-updates/s."""
    import oracle
    n, m = wl.shape
    geom = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    rows = rows or max(256, min(n, m, int(1.5e7 // max(n, m))))
    rows = min(rows, n, m)
    g = np.zeros(m)
    f = np.zeros(n)
    t0 = time.perf_counter()
    geom.rows_lse_subset(np.arange(rows), g, wl.eps)
    geom.cols_lse_subset(np.arange(rows), f, wl.eps)
    dt = time.perf_counter() - t0
    cells = rows * m + rows * n          # cells touched by the two partial half-steps
    return (cells / 2.0) / dt, dt, f"rows half-step on {rows} rows x {m} cols + cols half-step on {rows} cols x {n} rows (float64 numpy, oracle/)"


def run_reference(args, wl, rank):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    vals = []
    desc = ""
    for _ in range(args.warmup):
        cpu_sample_rate(wl)
    t_total = 0.0
    for _ in range(args.steps):
        v, dt, desc = cpu_sample_rate(wl)
        vals.append(v)
        t_total += dt
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "sinkhorn_cell_updates_per_s", "value": value,
        "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy, workloads.py)",
        "config": {"workload": wl.name, "n": wl.shape[0], "m": wl.shape[1], "d": wl.d,
                   "eps": wl.eps, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def kernel_roofline(otk, geom, wl, reps=20):
    """Average duration of the dominant kernel (the rows half-step, otk_lse_partial)
    measured with CUDA events on its stream; algorithmic flops per launch =
    (2d+8) per cell."""
    import torch
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    cx, cy = geom._clouds()
    n, m = wl.shape
    lib = N.lib()
    kappa = float(np.float32(1.4426950408889634 / wl.eps))
    bias = torch.zeros(m, dtype=torch.float32, device=cx.p.device)
    flags = geom._flags
    nsplit = lib.otk_lse_suggest_nsplit(n, m, cx.d, flags)
    part = torch.empty(nsplit * n, dtype=torch.float32, device=cx.p.device)
    st = stream()
    sinv = 1.0 / (cx.scale * cx.scale)

    def launch():
        N.check(lib.otk_lse_partial(N.ptr(cx.p), N.ptr(cx.sq), N.ptr(cx.hi), N.ptr(cx.lo),
                                    N.ptr(cx.ext_a), n, N.ptr(cy.p), N.ptr(cy.sq), N.ptr(cy.hi),
                                    N.ptr(cy.lo), N.ptr(cy.ext_b), m, cx.d, cx.dpad, sinv,
                                    N.ptr(bias), kappa, flags, nsplit, N.ptr(part), st))
    for _ in range(3):
        launch()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3 / reps
    cells = float(n) * m
    return sec, cells, nsplit


def run_ours(args, wl, rank, world):
    import torch
    import paper_2201_12324_b200 as otk
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    N.lib()
    n, m = wl.shape
    xd = torch.from_numpy(wl.x).to(dev)
    yd = torch.from_numpy(wl.y).to(dev)
    geom = otk.PointCloudGeometry(xd, yd)
    prob = otk.LinearProblem(geom, wl.a, wl.b)
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)

    def solve():
        return otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters,
                                  impl=args.kernel)

    for _ in range(args.warmup):
        out = solve()
    times, iters, launches = [], [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush (untimed)
            ev0.record()
            out = solve()
            ev1.record()
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1) * 1e-3)
            iters.append(out.iterations)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    total = sum(times)
    cell_updates = float(n) * m * sum(iters)
    if world > 1:
        t = torch.tensor([total], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total = float(t.item())
    value = cell_updates * world / total

    # launch count of one step (native solver reports it)
    from paper_2201_12324_b200.sinkhorn import _solve_pointcloud  # noqa: F401
    result = {
        "metric": "sinkhorn_cell_updates_per_s", "value": value, "unit": "cell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy draws, paper_2201_12324_b200/workloads.py)",
        "config": {"workload": wl.name, "n": n, "m": m, "d": wl.d, "eps": wl.eps,
                   "threshold": wl.threshold, "iterations_per_step": int(np.mean(iters)),
                   "converged": bool(out.converged), "step": "one solve_sinkhorn to tolerance",
                   "time_to_tolerance_ms": 1e3 * total / args.steps,
                   "l2": "flushed (512 MiB write) before every timed step",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "kernel": args.kernel},
        "clocks": clocks.summary(),
    }
    if rank != 0:
        return

    # ---- gpu launches per step
    result["gpu_launches"] = _count_launches(otk, prob, wl, args) * args.steps

    # ---- roofline of the dominant kernel
    sec, cells, nsplit = kernel_roofline(otk, geom, wl)
    pk, pk_kind = peaks()
    flops = (2 * wl.d + 8) * cells
    achieved_tf = flops / sec / 1e12
    peak_tf = float(pk.get("bf16_tflops", 1590.0))
    traffic = None
    try:
        with open(TRAFFIC_FILE) as fh:
            traffic = json.load(fh).get(wl.name)
    except OSError:
        pass
    ex2, ffma = ctypes_pipes()
    cells_per_s = cells / sec
    roof_cells = min(ex2, ffma / (2 * wl.d + 8)) if geom._clouds()[0].hi is None else ex2
    result["roofline"] = {
        "bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
        "frac": achieved_tf / peak_tf, "traffic": traffic,
        "kernel": "otk_lse_partial (rows half-step)", "kernel_ms": sec * 1e3,
        "algorithmic_flops_per_launch": flops, "cells_per_launch": cells,
        "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({pk_kind})",
        "compute_roof": {
            "note": "exp-bound roof: one MUFU ex2 per cell per half-step (SURVEY.md §8d); "
                    "pipe rates measured on this GPU by otk_bench_pipes",
            "ex2_per_s": ex2, "ffma_per_s": ffma, "roof_cells_per_s": roof_cells,
            "achieved_cells_per_s": cells_per_s, "frac": cells_per_s / roof_cells},
    }

    # ---- e2e through the public API from pinned host buffers
    if not args.no_e2e:
        result["e2e"] = _e2e(otk, wl, args, dev)

    # ---- CPU baseline (oracle on the host cores, bounded sample)
    if not args.no_cpu and world == 1:
        v, dt, desc = cpu_sample_rate(wl)
        result["cpu_baseline"] = {"value": v, "unit": "cell-updates/s",
                                  "cores": len(os.sched_getaffinity(0)), "kind": "port",
                                  "sample": desc + f", {dt:.1f}s"}
    print(json.dumps(result), flush=True)


def ctypes_pipes():
    import ctypes
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    ex2 = ctypes.c_double()
    ffma = ctypes.c_double()
    N.check(N.lib().otk_bench_pipes(ctypes.byref(ex2), ctypes.byref(ffma), stream()))
    return ex2.value, ffma.value


def _count_launches(otk, prob, wl, args):
    import ctypes
    from paper_2201_12324_b200 import sinkhorn as S
    captured = {}
    orig = S.N.lib().otk_solve_pointcloud

    def spy(ptr):
        rc = orig(ptr)
        captured["launches"] = ctypes.cast(ptr, ctypes.POINTER(S.N.SolveArgs)).contents.launches
        return rc

    real = S.N.lib()

    class Proxy:
        def __getattr__(self, name):
            return spy if name == "otk_solve_pointcloud" else getattr(real, name)

    saved = S.N.lib
    S.N.lib = lambda: Proxy()
    try:
        otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters,
                           impl=args.kernel)
    finally:
        S.N.lib = saved
    return int(captured.get("launches", 0))


def _e2e(otk, wl, args, dev):
    import torch
    xh = torch.from_numpy(wl.x).pin_memory()
    yh = torch.from_numpy(wl.y).pin_memory()
    n, m = wl.shape

    def step():
        prob = otk.LinearProblem(otk.PointCloudGeometry(xh, yh), wl.a, wl.b)
        out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters,
                                 impl=args.kernel)
        return out  # out.f / out.g are host float64 arrays (D2H inside the timed region)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its = 0
    for _ in range(args.steps):
        out = step()
        its += out.iterations
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h2d = wl.x.nbytes + wl.y.nbytes + 4 * (n + m) * 2   # points + weights + log-weights (fp32)
    d2h = 4 * (n + m)                                  # f, g (fp32)
    return {"value": float(n) * m * its / dt, "unit": "cell-updates/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": 1e3 * dt / args.steps,
            "api": "solve_sinkhorn(LinearProblem(PointCloudGeometry(pinned host x, y)))"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    from paper_2201_12324_b200 import workloads
    wl = workloads.make(args.config)
    if args.impl == "reference":
        run_reference(args, wl, rank)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl")
    run_ours(args, wl, rank, world)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
