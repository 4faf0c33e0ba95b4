"""Benchmark: Sinkhorn cell-updates/s (n*m*iters/s) and time-to-tolerance.

Default workload = BASELINE.json configs[3] (cfg4: n = 262144, m = 131072,
d = 128, non-uniform weights, eps = 0.05 x subsample mean, tolerance 1e-3):
the largest configuration that fits one GPU, the one the north star's
8-GPU scaling target names.  One STEP = one fixed-iteration solve (--iters,
default 100: threshold 1e-300, the reference's check every 10 iterations
still runs) on inputs already resident in HBM; value = n*m*iterations / step
time -- SURVEY.md §8d: "throughput comes from fixed-iteration runs".  The
time-to-tolerance (the workload's own threshold and max_iters) is timed
separately under the same rules, INCLUDING the prep of the geometry (norms,
split planes) and the on-device eps estimate (config.time_to_tolerance_ms);
--iters 0 makes the tolerance solve the step.  L2 is flushed (512 MiB write)
before every timed step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config k]

--gpus N > 1 without torchrun: bench.py re-launches itself under
``torch.distributed.run`` with N ranks (127.0.0.1) and asserts the world size.
N > 1 (one rank per GPU, NCCL): the row-sharded solver
(paper_2201_12324_b200/sharded.py) on the SAME problem -- x
split in N row shards, the g half-step's m partials per rank pushed to every
rank over NVLink peer memory (csrc/p2p.cu) -- so the scaling is strong;
value = n*m*iters / max-over-ranks step time.  --config 3 runs the batched
materialised path (512 problems of 512^2).

``--impl reference`` times the reference's CPU algorithm (the float64 numpy
restatement under oracle/; the reference itself is pure Python/numpy) on a
bounded sample of the same workload on rank 0's host cores.  Both arms print
the same ``config`` object; run-specific facts go under ``run``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "roofline_traffic.json")
METRIC = "sinkhorn_cell_updates_per_s"
UNIT = "cell-updates/s"
DATA = "synthetic (seeded numpy draws with the BASELINE.json shapes/distributions, workloads.py)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--plumbing", action="store_true",
                    help="(test) launch N ranks over gloo, check the world size, print it and exit")
    ap.add_argument("--iters", type=int, default=100,
                    help="timed step = a fixed-iteration solve of this many iterations "
                         "(SURVEY.md §8d: throughput from fixed-iteration runs); 0 = the "
                         "tolerance solve.  Time-to-tolerance is measured and reported either way")
    return ap.parse_args()


def solve_kw(wl, iters):
    """Solver arguments of a step: fixed `iters` iterations (fixed_iters: the checks
    run at the reference's cadence and are recorded but never stop the loop -- the
    float32 iterates of the small configs reach an exact fixed point, marginal
    error 0.0, before 100 iterations) or, with iters == 0, the workload's tolerance run."""
    if iters and iters > 0:
        return {"threshold": 1e-300, "max_iters": int(iters), "fixed_iters": True}
    return {"threshold": wl.threshold, "max_iters": wl.max_iters}


def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


def traffic_for(name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(TRAFFIC_FILE) as fh:
            v = json.load(fh).get(name)
        return float(v) if v is not None else None
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ clocks
_SAMPLER_SRC = r"""
import json, sys, time
import pynvml
idx, period = int(sys.argv[1]), float(sys.argv[2])
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(idx)
out = []
sys.stdout.write("ready\n"); sys.stdout.flush()
import select
while True:
    r, _, _ = select.select([sys.stdin], [], [], 0)
    if r:
        break
    out.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
    time.sleep(period)
sys.stdout.write(json.dumps(out) + "\n"); sys.stdout.flush()
"""


class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) while the timed region runs,
    every `period` s, from a SEPARATE process: a sampling thread in this
    process would contend with the timed host code (GIL, driver locks) --
    measured on cfg1, a 2 ms in-process sampler stretched a 0.8 ms solve to
    4.3 ms.  Only the samples taken inside [enter, exit] are kept."""

    REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index=0, period=None):
        import subprocess
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.proc = None
        if period is None:
            period = float(os.environ.get("OTK_CLOCK_PERIOD", "0.01"))
        self.period = period
        try:
            if period <= 0:
                raise RuntimeError("sampling disabled")
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(index), str(period)],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            if self.proc.stdout.readline().strip() != "ready":
                raise RuntimeError("clock sampler did not start")
        except Exception:  # noqa: BLE001
            self.proc = None

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *exc):
        self.t1 = time.time()
        if self.proc is None:
            return
        try:
            out, _ = self.proc.communicate("stop\n", timeout=30)
            rows = json.loads(out.strip().splitlines()[-1])
        except Exception:  # noqa: BLE001
            self.proc.kill()
            return
        inside = [r for r in rows if self.t0 <= r[0] <= self.t1]
        if not inside and rows:  # a region shorter than one period: the nearest sample
            inside = [min(rows, key=lambda r: abs(r[0] - 0.5 * (self.t0 + self.t1)))]
        for _, mhz, mask in inside:
            self.samples.append(mhz)
            for bit, name in self.REASONS.items():
                if mask & bit:
                    self.reasons.add(name)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "sampler": f"separate process, NVML every {self.period * 1e3:g} ms"}


# ------------------------------------------------------------------ CPU reference arm
def cpu_sample_rate(wl, budget_s=10.0):
    """The oracle (float64 numpy restatement of the reference) on a bounded sample of
    the workload, repeated until ~budget_s of CPU work: online configs run a rows
    half-step on R rows and a cols half-step on R columns, each reducing over the
    FULL other axis (= R*(n+m)/2 cell-updates); the batched config runs full
    iterations of a few of its problems.  Returns (cell-updates/s, seconds, desc)."""
    import oracle
    t0 = time.perf_counter()
    cells, reps = 0.0, 0
    if wl.materialised:
        B = wl.x.shape[0]
        k = min(B, 4)
        probs = []
        for p in range(k):
            geom = oracle.PointCloudOracle(wl.x[p].astype(np.float64), wl.y[p].astype(np.float64))
            probs.append((oracle.DenseOracle(geom.cost_matrix()), geom.shape, float(wl.eps[p])))
        t0 = time.perf_counter()
        while reps == 0 or time.perf_counter() - t0 < budget_s:
            for dense, (n, m), e in probs:
                g = np.zeros(m)
                f = -dense.apply_lse_kernel(np.zeros(n), g, e, "rows")
                g = -dense.apply_lse_kernel(f, np.zeros(m), e, "cols")
                cells += n * m
            reps += 1
        dt = time.perf_counter() - t0
        return cells / dt, dt, (f"{reps} x one full iteration of {k} of {B} problems "
                                "(DenseGeometry, float64 numpy)")
    n, m = wl.shape
    geom = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    rows = min(n, m, max(256, int(1e8 // max(n, m))))
    t0 = time.perf_counter()
    while reps == 0 or time.perf_counter() - t0 < budget_s:
        geom.rows_lse_subset(np.arange(rows), np.zeros(m), wl.eps)
        geom.cols_lse_subset(np.arange(rows), np.zeros(n), wl.eps)
        cells += rows * (n + m) / 2.0
        reps += 1
    dt = time.perf_counter() - t0
    return cells / dt, dt, (f"{reps} x (rows half-step on {rows} rows x {m} cols + cols "
                            f"half-step on {rows} cols x {n} rows), float64 numpy (oracle/)")


def cpu_cores():
    return len(os.sched_getaffinity(0))


def run_reference(args, wl, rank):
    if rank != 0:
        return
    # each step is a bounded sample; the budget per step keeps the whole K-step run at
    # about two minutes of CPU samples (15 s per step at the default K = 5)
    budget = min(15.0, max(3.0, 120.0 / max(args.steps, 1)))
    for _ in range(args.warmup):
        cpu_sample_rate(wl, budget_s=min(2.0, budget))
    vals, t_total, desc = [], 0.0, ""
    for _ in range(args.steps):
        v, dt, desc = cpu_sample_rate(wl, budget_s=budget)
        vals.append(v)
        t_total += dt
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(wl),
        "run": {"parallelism": "cpu (oracle port of the reference, rank 0's host cores)",
                "iters_per_sample": "see cpu_baseline.sample"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(wl):
    """The workload only -- identical in both arms (the driver compares them)."""
    n, m = wl.shape
    cfg = {"workload": wl.name, "n": n, "m": m, "d": wl.d, "threshold": wl.threshold,
           "max_iters": wl.max_iters, "inner_iters": wl.inner_iters,
           "weights": "uniform" if wl.a is None else "non-uniform (U(0.5,1.5), normalised)",
           "l2": "flushed (512 MiB write) before every timed step (GPU arm)"}
    if wl.materialised:
        cfg["batch"] = int(wl.x.shape[0])
        cfg["eps"] = "per problem: 0.05 x exact mean cost"
    else:
        cfg["eps"] = wl.eps
    return cfg


# ------------------------------------------------------------------ device timing helpers
def event_time(fn, reps, stream_ptr=None):
    """Mean seconds of fn() over reps, CUDA events on torch's current stream
    (the stream every library call in fn is launched on)."""
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def pipes():
    import ctypes
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    ex2, ffma = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().otk_bench_pipes(ctypes.byref(ex2), ctypes.byref(ffma), stream()))
    return ex2.value, ffma.value


def online_roofline(geom, wl, reps=10):
    """Dominant kernel of the online path: one rows half-step as the solver runs
    it in steady state -- otk_lse_step with the row anchors of the previous
    half-step (anchored tcgen05 kernel + finalize + the idle repair check), or
    otk_lse_partial + finalize on the FP32 path -- timed with CUDA events on its
    stream.  Algorithmic work per cell: 2d dot-product flops +
    8 epilogue flops + 1 exp."""
    import torch
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    cx, cy = geom._clouds()
    n, m = geom.shape
    lib = N.lib()
    kappa = float(np.float32(1.4426950408889634 / wl.eps))
    dev = cx.p.device
    bias = torch.zeros(m, dtype=torch.float32, device=dev)
    flags = geom._flags
    nsplit = lib.otk_lse_suggest_nsplit(n, m, cx.d, flags)
    part = torch.empty(nsplit * n, dtype=torch.float32, device=dev)
    sinv = 1.0 / (cx.scale * cx.scale)
    tc = cx.hi is not None and not (flags & N.OTK_IMPL_SIMT)
    anchored = bool(lib.otk_lse_step_anchored(n, m, cx.d, flags))
    base = torch.full((n,), float(np.log(1.0 / n)), dtype=torch.float32, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    anchor = torch.empty(n, dtype=torch.float32, device=dev)
    rep = torch.empty(lib.otk_lse_step_workspace_bytes(n), dtype=torch.uint8, device=dev)

    def step(fl):
        N.check(lib.otk_lse_step(N.ptr(cx.p), N.ptr(cx.sq), N.ptr(cx.hi), N.ptr(cx.lo),
                                 N.ptr(cx.ext_a), n, N.ptr(cy.p), N.ptr(cy.sq), N.ptr(cy.hi),
                                 N.ptr(cy.lo), N.ptr(cy.ext_b), m, cx.d, cx.dpad, sinv,
                                 N.ptr(bias), kappa, fl, nsplit, N.ptr(part), N.ptr(base),
                                 N.OTK_FIN_SOLVER, float(wl.eps), kappa, N.ptr(out), None, None, 0,
                                 N.ptr(anchor), N.ptr(rep), None, stream()))

    step(flags | N.OTK_ANCHOR_INIT)  # anchors of the "previous" half-step

    def launch():
        step(flags)
    for _ in range(3):
        launch()
    sec = event_time(launch, reps)
    cells = float(n) * m
    pk, pk_kind = peaks()
    ex2, ffma = pipes()
    cps = cells / sec
    d = wl.d
    if tc:
        peak = float(pk.get("bf16_tflops", 1590.0)) / 3.0
        achieved = 2.0 * d * cps / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak,
                "peak_note": f"{pk_kind} dense bf16 / 3: the 3-product split-fp16 contraction "
                             "that carries fp32 accuracy (SURVEY.md §8d P_dot)",
                "achieved_note": "2d dot-product flops per cell / kernel time "
                                 "(the 8 epilogue flops + 1 exp run on FP32/MUFU)"}
    else:
        achieved = (2.0 * d + 8.0) * cps / 1e12
        peak = 2.0 * ffma / 1e12
        roof = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "peak_note": "FP32 FFMA rate measured on this GPU x 2"}
    roof.update({
        "traffic": traffic_for(wl.name),
        "kernel": ("otk_lse_step, anchored (lse_tc FIX kernel + finalize + idle repair check)"
                   if anchored else "otk_lse_step (rows half-step: partial + finalize)"),
        "kernel_ms": sec * 1e3, "cells_per_launch": cells,
        "algorithmic_flops_per_launch": (2.0 * d + 8.0) * cells,
        "pipes": {"ex2_per_s": ex2, "ffma_per_s": ffma, "cells_per_s": cps,
                  "mufu_frac": cps / ex2,
                  "note": "one MUFU ex2 per cell per half-step; tcgen05.ld reads 4 B of TMEM "
                          "per cell (~64 B/clk/SM) -- the measured binding resource (profiles/)"},
    })
    return roof


def small_roofline(value, step_s, wl):
    """The whole solve is ONE persistent kernel (solve_small.cu, problems that
    fit in shared memory -- cfg1): its roof is MUFU ex2, 2 exps per
    cell-update (one per cell per half-step; cfg1 is MUFU-bound),
    achieved = 2 x cell-updates/s of the timed steps (one launch per step, so
    the kernel time is the step time), peak = the ex2 rate measured on this GPU."""
    ex2, ffma = pipes()
    achieved = 2.0 * value
    return {"bound": "mufu", "achieved": achieved / 1e9, "peak": ex2 / 1e9, "unit": "Gex2/s",
            "frac": achieved / ex2, "traffic": traffic_for(wl.name),
            "kernel": "solve_small_kernel (whole solve, one launch)", "kernel_ms": step_s * 1e3,
            "cells_per_launch": float(wl.x.shape[0]) * wl.y.shape[0],
            "peak_note": "MUFU ex2 rate measured on this GPU (csrc/pipes.cu)",
            "achieved_note": "the log-domain formulation's 2 ex2 per cell-update x cell-updates/s of "
                             "the timed steps (SURVEY.md 8d's unit of work); the stored-kernel "
                             "half-steps take the exps once per build and then do one FFMA per cell, "
                             "and the kernel is latency-bound (half-step exchange, reductions: "
                             "tools/small_trace.py), not MUFU-bound",
            "pipes": {"ex2_per_s": ex2, "ffma_per_s": ffma}}


def dense_roofline(C, wl, reps=3):
    """Dominant kernel of the batched materialised path: the one-launch batched
    solve (otk_solve_dense_batched: K3c by default, K3p with OTK_DENSE_KERNEL=cta),
    timed with CUDA events on its stream.  K3c's roof is the shared-memory read
    rate: 4 B of its stored kernel per cell per half-step, 2*iters + 1
    half-steps per problem (the fused check's extra row pass included); the
    HBM streaming-equivalent rate is reported beside it.  K3p's roof is HBM."""
    import ctypes
    import torch
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    B, n, m = C.shape
    dev = C.device
    lib = N.lib()
    a = torch.full((B, n), 1.0 / n, dtype=torch.float32, device=dev)
    b = torch.full((B, m), 1.0 / m, dtype=torch.float32, device=dev)
    la, lb = torch.full_like(a, -float(np.log(n))), torch.full_like(b, -float(np.log(m)))
    eps32 = torch.as_tensor(np.asarray(wl.eps, dtype=np.float32), device=dev)
    eps64 = torch.as_tensor(np.asarray(wl.eps, dtype=np.float64), device=dev)
    mc = wl.max_iters // wl.inner_iters + 2
    f, g = torch.empty((B, n), device=dev), torch.empty((B, m), device=dev)
    errs = torch.empty((B, mc), dtype=torch.float64, device=dev)
    duals = torch.empty_like(errs)
    state = torch.zeros((B, 5), dtype=torch.int32, device=dev)

    def launch():
        N.check(lib.otk_solve_dense_batched(
            N.ptr(C), B, n, m, N.ptr(a), N.ptr(b), N.ptr(la), N.ptr(lb), N.ptr(eps32), N.ptr(eps64),
            None, float(wl.threshold), int(wl.max_iters), int(wl.inner_iters), mc, N.ptr(f), N.ptr(g),
            N.ptr(errs), N.ptr(duals), N.ptr(state), 0, stream()))
    for _ in range(2):
        launch()
    sec = event_time(launch, reps)
    iters = state.cpu().numpy()[:, 1].astype(np.float64)
    nbytes = 4.0 * n * m * float(np.sum(2 * iters + 1))
    pk, pk_kind = peaks()
    gbs = nbytes / sec / 1e9
    read_gbs = ctypes.c_double()
    N.check(lib.otk_bench_read(N.ptr(C), int(4 * B * n * m), ctypes.byref(read_gbs), stream()))
    cluster = os.environ.get("OTK_DENSE_KERNEL", "cluster") != "cta"
    ex2, _ = pipes()
    exps = float(n) * m * float(np.sum(2 * iters + 1))
    if not cluster:  # K3p streams C from L2/HBM every half-step: the byte roof binds
        return {"bound": "hbm", "achieved": gbs, "peak": float(pk["hbm_gbs"]), "unit": "GB/s",
                "frac": gbs / float(pk["hbm_gbs"]), "traffic": traffic_for(wl.name),
                "kernel": "otk_solve_dense_batched (K3p: one CTA per problem streaming C, one launch)",
                "kernel_ms": sec * 1e3, "algorithmic_bytes_per_launch": nbytes, "peak_note": pk_kind,
                "read_only_gbs": read_gbs.value, "read_only_frac": gbs / read_gbs.value,
                "mufu": {"ex2_per_s": exps / sec, "peak_ex2_per_s": ex2, "frac": exps / sec / ex2}}
    # K3c keeps each problem's stabilised kernel resident in its cluster's shared
    # memory (built from C, read from HBM ONCE per solve: traffic) and runs every
    # half-step as an FP32 matrix-vector product over it: its roof is the
    # shared-memory read rate, 4 B of kernel per cell per half-step
    smem = ctypes.c_double()
    N.check(lib.otk_bench_smem(ctypes.byref(smem), stream()))
    sbytes = 4.0 * n * m * float(np.sum(2 * iters + 1))
    return {"bound": "smem", "achieved": sbytes / sec / 1e9, "peak": smem.value / 1e9, "unit": "GB/s",
            "frac": sbytes / sec / smem.value, "traffic": traffic_for(wl.name),
            "kernel": ("otk_solve_dense_batched (K3c: stabilised kernel resident in a cluster's shared "
                       "memory, FP32 matrix-vector half-steps, one launch)"),
            "kernel_ms": sec * 1e3, "algorithmic_bytes_per_launch": sbytes,
            "peak_note": "shared-memory LDS.128 read rate measured on this GPU (csrc/pipes.cu otk_bench_smem)",
            "achieved_note": "4 B of the stored kernel per cell per half-step (2*iters + 1 half-steps per "
                             "problem) / kernel time",
            "hbm_streaming_equivalent": {
                "gbs": gbs, "hbm_peak_gbs": float(pk["hbm_gbs"]), "frac": gbs / float(pk["hbm_gbs"]),
                "read_only_gbs": read_gbs.value,
                "note": "what a kernel streaming 4 B of C per cell per half-step from HBM would have to "
                        "move / time"},
            "mufu": {"ex2_per_s_log_domain_equivalent": exps / sec, "peak_ex2_per_s": ex2,
                     "note": "the log-domain formulation's one ex2 per cell per half-step / time; the "
                             "scaling domain takes the exps once per kernel build"}}


# ------------------------------------------------------------------ our arm
def timed_steps(solve, steps, dev, flush):
    """Barrier-free local timing of `steps` solves, CUDA events, L2 flushed before each."""
    import torch
    times, outs = [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for _ in range(steps):
        flush.fill_(1.0)
        ev0.record()
        out = solve()
        ev1.record()
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1) * 1e-3)
        outs.append(out)
    return times, outs


def run_ours(args, wl, rank, world):
    import torch
    import paper_2201_12324_b200 as otk
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200 import workloads
    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    N.lib()
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    n, m = wl.shape

    kw_step = solve_kw(wl, args.iters)
    kw_tol = solve_kw(wl, 0)
    tol_note = "one tolerance solve from device-resident points"
    exchange_note = None
    if wl.materialised:
        xd = torch.from_numpy(wl.x).to(dev)
        yd = torch.from_numpy(wl.y).to(dev)

        def make_solve(kw):
            return lambda: otk.solve_sinkhorn_batched(xd, yd, wl.eps, **kw)

        solve_tol = make_solve(kw_tol)
        tol_note += " (cost build included; per-problem eps given)"

        def cells_of(outs):
            return float(n) * m * float(np.sum(outs.iterations))
        parallelism = "single GPU, batched"
    elif world > 1:
        from paper_2201_12324_b200.sharded import TorchComm, shard_rows
        comm = TorchComm()
        lo, hi = shard_rows(n, world, rank)
        xd = torch.from_numpy(wl.x[lo:hi]).to(dev)
        yd = torch.from_numpy(wl.y).to(dev)
        a_loc = None if wl.a is None else wl.a[lo:hi]
        ix, iy = workloads.subsample_rows(n, m, wl.eps_subsample_seed or 0)
        x_sub = torch.from_numpy(wl.x[ix] if wl.eps_subsample_seed is not None else wl.x).to(dev)

        exchange = os.environ.get("OTK_EXCHANGE", "auto")

        def new_problem():
            return otk.ShardedProblem(xd, yd, a_loc, wl.b, x_is_local=True, n_total=n, comm=comm,
                                      impl=args.kernel, exchange=exchange)
        sprob = new_problem()
        exchange_note = None
        if sprob.exchange == "p2p":
            # the peer-memory exchange must reproduce the NCCL all-gather path bit for
            # bit on a short solve before it is timed; otherwise every rank falls back
            ok = 1.0
            try:
                p_out = sprob.solve(wl.eps, threshold=1e-300, max_iters=3)
                c_out = otk.ShardedProblem(xd, yd, a_loc, wl.b, x_is_local=True, n_total=n, comm=comm,
                                           impl=args.kernel, exchange="collective").solve(
                    wl.eps, threshold=1e-300, max_iters=3)
                ok = float(np.array_equal(p_out.g, c_out.g) and np.array_equal(p_out.f_local, c_out.f_local))
            except Exception as exc:  # noqa: BLE001 -- reported in the JSON line, then the fallback
                exchange_note = f"peer exchange failed its check ({type(exc).__name__}: {exc})"
                ok = 0.0
            flag = torch.tensor([ok], device=dev)
            torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
            if flag.item() < 1.0:
                exchange = "collective"
                os.environ["OTK_EXCHANGE"] = "collective"  # the e2e leg too
                exchange_note = exchange_note or "peer exchange differed from the all-gather path"
                sprob = new_problem()
            else:
                exchange_note = "peer exchange verified bitwise against the NCCL all-gather path (3 iterations)"

        def make_solve(kw):
            def solve():
                return sprob.solve(wl.eps, **kw)
            solve.sharded_problem = sprob
            return solve

        def solve_tol():
            sp = new_problem()
            sub = wl if wl.eps_subsample_seed is None else \
                workloads.Workload(wl.name, wl.x, wl.y, None, None, wl.eps, wl.threshold,
                                   wl.max_iters, eps_scale=wl.eps_scale)
            e = workloads.estimate_eps_device(sub, x_sub, yd[torch.as_tensor(iy, device=dev)]
                                              if wl.eps_subsample_seed is not None else yd)
            return sp.solve(e, **kw_tol)
        tol_note += " (shard prep + on-device eps estimate included)"

        def cells_of(out):
            return float(n) * m * out.iterations
        parallelism = (f"row-sharded x{world} (native loop: g half-step partials pushed over NVLink "
                       "peer memory by the half-step's last kernel, check sums exchanged on the "
                       "device, CUDA-graph check periods)" if sprob.loop == "native" else
                       f"row-sharded x{world} ({sprob.exchange} exchange per g half-step, "
                       "Python loop)")
    else:
        xd = torch.from_numpy(wl.x).to(dev)
        yd = torch.from_numpy(wl.y).to(dev)
        geom = otk.PointCloudGeometry(xd, yd)
        prob = otk.LinearProblem(geom, wl.a, wl.b)

        def make_solve(kw):
            return lambda: otk.solve_sinkhorn(prob, wl.eps, impl=args.kernel, **kw)

        def solve_tol():
            g2 = otk.PointCloudGeometry(xd, yd)
            e = workloads.estimate_eps_device(wl, xd, yd)
            return otk.solve_sinkhorn(otk.LinearProblem(g2, wl.a, wl.b), e, impl=args.kernel,
                                      **kw_tol)
        tol_note += " (geometry prep + on-device eps estimate included)"

        def cells_of(out):
            return float(n) * m * out.iterations
        parallelism = "single GPU"
    solve = make_solve(kw_step)

    # the dominant kernel, timed alone BEFORE the long timed region (the burst
    # peak applies; after minutes of solves the part sits at its power cap)
    roofline = None
    if rank == 0:
        if wl.materialised:
            C = torch.empty((wl.x.shape[0], n, m), dtype=torch.float32, device=dev)
            N.check(N.lib().otk_dense_cost(N.ptr(xd), N.ptr(yd), wl.x.shape[0], n, m, wl.d, 0,
                                           N.ptr(C), None, torch.cuda.current_stream().cuda_stream))
            roofline = dense_roofline(C, wl)
            del C
        elif world == 1:
            roofline = online_roofline(geom, wl)
        else:
            roofline = online_roofline(otk.PointCloudGeometry(xd, yd), wl)
            roofline["note"] = "rank 0's shard (n/N rows x m)"
            roofline["traffic"] = None  # the committed ncu capture is single-GPU
        roofline["timed"] = "alone, before the timed solves (burst peak)"
    if world > 1:
        torch.distributed.barrier()

    # warm-up: at least W steps and at least ~1 s of steps (clocks, caches, allocator)
    t_w, n_w = time.perf_counter(), 0
    while True:
        solve()
        n_w += 1
        more = n_w < args.warmup or time.perf_counter() - t_w < 1.0
        if world > 1:  # every rank runs the same number of (collective) solves
            flag = torch.tensor([1.0 if more else 0.0], device=dev)
            torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MAX)
            more = flag.item() > 0.0
        if not more:
            break
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        times, outs = timed_steps(solve, args.steps, dev, flush)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total = float(t.item())
    cell_updates = sum(cells_of(o) for o in outs)
    value = cell_updates / total

    def summary(o):
        its = int(np.max(o.iterations)) if wl.materialised else o.iterations
        cv = bool(np.all(o.converged)) if wl.materialised else bool(o.converged)
        nchk = int(np.max([len(o[k].errors) for k in range(len(o.iterations))])) \
            if wl.materialised else len(o.errors)
        return its, cv, nchk
    iters, conv, _ = summary(outs[-1])
    # time-to-tolerance: the workload's own threshold / max_iters, same timing rules,
    # prep and eps estimate inside the timed call
    for _ in range(2):
        solve_tol()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_tol, o_tol = timed_steps(solve_tol, args.steps, dev, flush)
    tt = sum(t_tol)
    if world > 1:
        t = torch.tensor([tt], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tt = float(t.item())
    tol_ms = 1e3 * tt / args.steps
    tol_iters, tol_conv, tol_checks = summary(o_tol[-1])
    # the same tolerance solve on the already-prepared problem (solver time alone)
    solve_only = make_solve(kw_tol)
    for _ in range(2):
        solve_only()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_so, _ = timed_steps(solve_only, args.steps, dev, flush)
    tso = sum(t_so)
    if world > 1:
        t = torch.tensor([tso], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tso = float(t.item())
    step_desc = (f"one fixed {kw_step['max_iters']}-iteration solve (fixed_iters: convergence test off, checks every "
                 f"{wl.inner_iters} as in the reference; SURVEY.md §8d: throughput from "
                 "fixed-iteration runs), inputs resident in HBM" if args.iters
                 else "one complete solve to tolerance (inputs resident in HBM)")
    run = {"parallelism": parallelism, "iterations_per_step": iters, "converged": conv,
           "step_ms": [round(1e3 * t_, 4) for t_ in times],
           **({"exchange_check": exchange_note} if world > 1 and not wl.materialised else {}),
           "step": step_desc, "time_to_tolerance_ms": tol_ms,
           "time_to_tolerance_solve_only_ms": 1e3 * tso / args.steps, "tolerance_iterations": tol_iters,
           "tolerance_converged": tol_conv, "tolerance_checks": tol_checks,
           "time_to_tolerance_note": tol_note, "kernel": args.kernel}
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": n_w, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": DATA,
        "config": workload_config(wl), "run": run, "clocks": clocks.summary(),
    }

    # launches of our kernels per step (native solver count / sharded engine count)
    result["gpu_launches"] = count_launches(otk, wl, args, solve, world) * args.steps
    if rank == 0 and world == 1 and not wl.materialised and result["gpu_launches"] == args.steps:
        roofline = small_roofline(value, total / args.steps, wl)

    if not args.no_e2e:
        e2e = run_e2e(otk, wl, args, dev, world, rank)
        if e2e is not None:
            result["e2e"] = e2e
    if rank == 0:
        result["roofline"] = roofline
        if not args.no_cpu and world == 1:
            v, dt, desc = cpu_sample_rate(wl)
            # the reference's time for the same tolerance solve: its half-steps
            # (2 per iteration + 1 per check) at the measured CPU rate
            half_steps = 2.0 * tol_iters + tol_checks
            cpu_ttt = half_steps * 0.5 * float(n) * m * (wl.x.shape[0] if wl.materialised else 1) / v
            result["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                "sample": f"{desc}, {dt:.1f} s",
                "time_to_tolerance_s_extrapolated": cpu_ttt,
                "time_to_tolerance_note": (f"extrapolated: the GPU tolerance solve's {tol_iters} "
                                           f"iterations + {tol_checks} checks = {half_steps:.0f} "
                                           "half-steps at the sampled CPU rate")}
        print(json.dumps(result), flush=True)


def count_launches(otk, wl, args, solve, world):
    """Kernels of ours launched by one step: the native solver reports its count
    (graph nodes included); the sharded engine and the dense loop count theirs."""
    import ctypes
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200 import sinkhorn as S
    if wl.materialised:
        calls = {"n": 0}
        real = N.lib()

        class Counting:
            def __getattr__(self, name):
                fn = getattr(real, name)
                if not name.startswith("otk_") or name in ("otk_last_error", "otk_abi_version"):
                    return fn

                def wrapped(*a):
                    calls["n"] += 1
                    return fn(*a)
                return wrapped
        saved = S.N.lib
        S.N.lib = lambda: Counting()
        try:
            solve()
        finally:
            S.N.lib = saved
        return calls["n"]
    if world > 1:
        sp = solve.sharded_problem
        if sp.loop == "native":  # otk_solve_pointcloud_sharded reports its count (graph nodes incl.)
            solve()
            return int(sp.launches_last)
        eng = sp.engine
        before = eng.launches
        solve()
        return int(eng.launches - before)
    captured = {}
    real = N.lib()

    class Proxy:
        def __getattr__(self, name):
            if name == "otk_solve_pointcloud":
                def spy(ptr):
                    rc = real.otk_solve_pointcloud(ptr)
                    captured["launches"] = ctypes.cast(ptr, ctypes.POINTER(N.SolveArgs)).contents.launches
                    return rc
                return spy
            return getattr(real, name)
    saved = S.N.lib
    S.N.lib = lambda: Proxy()
    try:
        solve()
    finally:
        S.N.lib = saved
    return int(captured.get("launches", 0))


def run_e2e(otk, wl, args, dev, world, rank):
    """Same metric through the public API from pinned HOST buffers: every step
    copies its inputs host->device and reads the potentials back."""
    import torch
    kw = solve_kw(wl, args.iters)
    n, m = wl.shape
    if wl.materialised:
        xh = torch.from_numpy(wl.x).pin_memory()
        yh = torch.from_numpy(wl.y).pin_memory()

        def step():
            outs = otk.solve_sinkhorn_batched(xh, yh, wl.eps, **kw)
            assert outs.f.shape[0] == outs.g.shape[0]  # the potentials read back (D2H)
            return int(np.sum(outs.iterations))
        h2d = wl.x.nbytes + wl.y.nbytes
        d2h = 4 * (n + m) * wl.x.shape[0]
    elif world > 1:
        from paper_2201_12324_b200.sharded import TorchComm, shard_rows
        lo, hi = shard_rows(n, world, rank)
        xh = torch.from_numpy(wl.x[lo:hi]).pin_memory()
        yh = torch.from_numpy(wl.y).pin_memory()
        comm = TorchComm()

        def step():
            out = otk.solve_sinkhorn_sharded(xh, yh, wl.eps, None if wl.a is None else wl.a[lo:hi],
                                             wl.b, x_is_local=True, n_total=n,
                                             **kw,
                                             comm=comm, impl=args.kernel)
            return out.iterations
        h2d = (hi - lo) * wl.d * 4 + wl.y.nbytes + 8 * (hi - lo + m)
        d2h = 4 * (hi - lo + m)
    else:
        xh = torch.from_numpy(wl.x).pin_memory()
        yh = torch.from_numpy(wl.y).pin_memory()

        def step():
            prob = otk.LinearProblem(otk.PointCloudGeometry(xh, yh), wl.a, wl.b)
            out = otk.solve_sinkhorn(prob, wl.eps, impl=args.kernel, **kw)
            return out.iterations  # out.f / out.g: float64 host arrays (D2H in the region)
        h2d = wl.x.nbytes + wl.y.nbytes + 4 * (n + m) * 2
        d2h = 4 * (n + m)
    # this leg repeats the whole workload through the public API: with second-long steps
    # (cfg4: 3.9 s) W warm-ups + K steps would double the run, so both are bounded by
    # time (>= 1 warm-up, >= 3 timed steps, ~10 s / ~40 s); every rank takes the same counts
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    est = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([est], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        est = float(t.item())
    n_warm = min(max(args.warmup - 1, 0), int(10.0 / max(est, 1e-6)))
    n_steps = min(args.steps, max(3, int(40.0 / max(est, 1e-6))))
    for _ in range(n_warm):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its = 0
    for _ in range(n_steps):
        its += step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": float(n) * m * its / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / n_steps, "steps": n_steps,
            "warmup": n_warm + 1,
            "api": "public API on pinned host arrays (H2D + D2H inside the timed region)"}


def local_device() -> int:
    """This rank's GPU.  OTK_BENCH_GLOO=1 (test only) puts every rank on GPU 0
    over gloo: the N > 1 code path can then be exercised on a one-GPU box
    without any kernel waiting on another rank's kernel (all exchanges go
    through host memory); its timings are meaningless."""
    if os.environ.get("OTK_BENCH_GLOO"):
        return 0
    return int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this same command as N ranks of
    ``torch.distributed.run`` (one node, 127.0.0.1) and return its exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def plumbing(args, rank, world):
    """(test) the multi-rank launch: gloo ranks agree on the world size."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"plumbing": True, "n_gpus": world, "gpus_arg": args.gpus,
                          "rank_sum": float(t.item())}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.plumbing:
        plumbing(args, rank, world)
        return
    from paper_2201_12324_b200 import workloads
    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args, workloads.make(args.config), rank)
        return
    wl = workloads.make(args.config)
    if world > 1:
        import torch
        torch.cuda.set_device(local_device())
        if os.environ.get("OTK_BENCH_GLOO"):  # multi-rank plumbing test on ONE GPU (see below)
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group(
                "nccl", device_id=torch.device("cuda", local_device()))
    try:
        run_ours(args, wl, rank, world)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
