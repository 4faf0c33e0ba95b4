"""Full-size golden fixtures from the UNMODIFIED reference, run over worker processes.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fullsize_golden.py cfg2 cfg5 cfg4 cfg3

The reference loop (`otkit.sinkhorn._sinkhorn_iterations`, sinkhorn.py:151-200)
runs as shipped in this process.  Its geometry is `PooledPointCloud`, which
answers `apply_lse_kernel` by calling the reference's own
`PointCloudGeometry.apply_lse_kernel` (geometry.py:336-354) on 256-aligned
row (or column) chunks in a fork pool.  Every output entry is reduced over its
full axis inside one reference call, with the same 256-row cost blocks
(`_cost_rows` / `_cost_cols`, geometry.py:278-292) as a single-process run, so
the result is the reference's (geometry.py:220-223: the block size never
changes results).  `reg_ot_cost` (sinkhorn.py:210-216) cannot materialise an
n x m plan at these sizes, so its two sums are evaluated with the reference's
expressions on 256-row cost blocks from the reference's `cost_matrix` and
added in block order (math.fsum); the dual then comes from the reference's
`_dual_objective` (sinkhorn.py:115-119).

Fixtures (inputs regenerate on the GPU box from workloads.py):

* ``full_cfg{2,5}_it{K}.npz`` / ``full_cfg4_it{K}.npz`` -- `solve_sinkhorn`
  with threshold 1e-300 and max_iters=K (the check at t == max_iters fires, so
  `errors` and `dual_trace` each hold one entry), f, g (float32-rounded to
  keep the files small; the parity gate is 1e-4), transport, dual.
* ``full_cfg{2,4,5}_tol.npz`` -- the same with the workload's own threshold
  and max_iters: the complete reference solve to tolerance at the BASELINE
  size (iterations, converged flag, f, g, errors, dual_trace, cost).
* ``full_cfg3_all.npz`` -- all 512 problems of cfg3 solved by the reference
  (DenseGeometry over the reference's cost_matrix, the workload's threshold and
  max_iters): iterations, converged, f, g, errors, dual_trace, transport, dual.
* ``conv_cfg{2,4,5}.npz`` (``conv`` mode, input = a GPU run's potentials saved
  by tools/dump_potentials.py) -- the reference's own check pass
  (sinkhorn.py:181-186) evaluated in float64 at the GPU's converged
  potentials: pins the converged flag the GPU reported.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import json  # noqa: E402
import math  # noqa: E402
import multiprocessing as mp  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import otkit  # noqa: E402  (reference, from PYTHONPATH)
import otkit.geometry as ogeo  # noqa: E402
import otkit.sinkhorn as osink  # noqa: E402

from paper_2201_12324_b200 import workloads  # noqa: E402

BLOCK = ogeo.DEFAULT_BLOCK_SIZE  # 256: the reference's row-block width
_X = None  # float64 point sets, inherited by the fork workers
_Y = None


def _lse_task(args):
    axis, lo, hi, f, g, eps = args
    if axis == "rows":
        geom = otkit.PointCloudGeometry(_X[lo:hi], _Y)
    else:
        geom = otkit.PointCloudGeometry(_X, _Y[lo:hi])
    return geom.apply_lse_kernel(f, g, eps, axis)


def _cost_task(args):
    """Partial (transport, mass) of sinkhorn.py:212-215 over rows [lo, hi), one
    reference cost block of BLOCK rows at a time."""
    lo, hi, f, g, eps = args
    parts = []
    for s in range(lo, hi, BLOCK):
        e = min(s + BLOCK, hi)
        geom = otkit.PointCloudGeometry(_X[s:e], _Y)
        cost = geom.cost_matrix(max_entries=(e - s) * _Y.shape[0])
        plan = np.exp((f[s - lo:e - lo, None] + g[None, :] - cost) / eps)
        parts.append((float((cost * plan).sum()), float(plan.sum())))
    return parts


class PooledPointCloud(ogeo.Geometry):
    """The reference's PointCloudGeometry (sqeucl), evaluated chunk-parallel."""

    def __init__(self, pool, n, m, chunk_blocks):
        self._shape = (n, m)
        self._epsilon_default = None
        self.pool = pool
        self.chunk = BLOCK * chunk_blocks
        self.calls = 0

    def apply_lse_kernel(self, f, g, eps=None, axis="rows"):
        ogeo._check_axis(axis)
        eps = self._resolve_eps(eps)
        n, m = self.shape
        f = ogeo._check_potential(f, n, "f")
        g = ogeo._check_potential(g, m, "g")
        size = n if axis == "rows" else m
        tasks = []
        for lo in range(0, size, self.chunk):
            hi = min(lo + self.chunk, size)
            if axis == "rows":
                tasks.append((axis, lo, hi, f[lo:hi], g, eps))
            else:
                tasks.append((axis, lo, hi, f, g[lo:hi], eps))
        t0 = time.perf_counter()
        out = np.concatenate(self.pool.map(_lse_task, tasks, chunksize=1))
        self.calls += 1
        print(f"  half-step {self.calls} ({axis}): {time.perf_counter() - t0:.1f}s", flush=True)
        return out

    def reg_ot_cost(self, out, prob):
        n, _ = self.shape
        tasks = [(lo, min(lo + self.chunk, n), out.f[lo:lo + self.chunk], out.g, out.eps)
                 for lo in range(0, n, self.chunk)]
        parts = [p for chunk in self.pool.map(_cost_task, tasks, chunksize=1) for p in chunk]
        transport = math.fsum(p[0] for p in parts)
        mass = math.fsum(p[1] for p in parts)
        dual = osink._dual_objective(out.f, out.g, prob.a, prob.b, out.eps, mass)
        return transport, dual, mass


def _pool(x, y, procs):
    global _X, _Y
    _X = np.asarray(x, np.float64)
    _Y = np.asarray(y, np.float64)
    return mp.get_context("fork").Pool(procs)


def full_solve(k, iters, procs, chunk_blocks):
    """iters=None: the workload's own tolerance run (threshold, max_iters)."""
    wl = workloads.make(k)
    n, m = wl.shape
    thr, mi = (wl.threshold, wl.max_iters) if iters is None else (1e-300, iters)
    print(f"cfg{k}: {n}x{m} d={wl.d} eps={wl.eps:.6g} threshold={thr} max_iters={mi}", flush=True)
    t0 = time.perf_counter()
    with _pool(wl.x, wl.y, procs) as pool:
        geom = PooledPointCloud(pool, n, m, chunk_blocks)
        prob = otkit.LinearProblem(geom, wl.a, wl.b)
        out = otkit.solve_sinkhorn(prob, wl.eps, threshold=thr, max_iters=mi,
                                   inner_iters=wl.inner_iters)
        t_solve = time.perf_counter() - t0
        transport, dual, mass = geom.reg_ot_cost(out, prob)
    dt = time.perf_counter() - t0
    print(f"cfg{k}: iters={out.iterations} errors={out.errors} dual_trace={out.dual_trace} "
          f"transport={transport!r} dual={dual!r} solve {t_solve:.0f}s total {dt:.0f}s", flush=True)
    save(f"full_cfg{k}_tol" if iters is None else f"full_cfg{k}_it{iters}", eps=np.array(wl.eps),
         threshold=np.array(thr), max_iters=np.array(mi),
         iterations=np.array(out.iterations), converged=np.array(out.converged),
         f=out.f.astype(np.float32), g=out.g.astype(np.float32),
         f_absmax=np.array(np.max(np.abs(out.f))), g_absmax=np.array(np.max(np.abs(out.g))),
         errors=out.errors, dual_trace=out.dual_trace, transport=np.array(transport),
         dual=np.array(dual), mass=np.array(mass), seconds=np.array(dt), procs=np.array(procs))


def _dense_task(k):
    wl = _CFG3
    x64 = wl.x[k].astype(np.float64)
    y64 = wl.y[k].astype(np.float64)
    n, m = x64.shape[0], y64.shape[0]
    cost = otkit.PointCloudGeometry(x64, y64).cost_matrix(max_entries=n * m)
    prob = otkit.LinearProblem(otkit.DenseGeometry(cost))
    out = otkit.solve_sinkhorn(prob, float(wl.eps[k]), threshold=wl.threshold,
                               max_iters=wl.max_iters, inner_iters=wl.inner_iters)
    old = ogeo.DEFAULT_DENSE_CAP
    ogeo.DEFAULT_DENSE_CAP = max(old, n * m)
    try:
        rc = otkit.reg_ot_cost(out, prob)
    finally:
        ogeo.DEFAULT_DENSE_CAP = old
    return (out.iterations, out.converged, out.f, out.g, out.errors, out.dual_trace,
            rc.transport_cost, rc.dual_objective)


_CFG3 = None


def cfg3_all(procs):
    global _CFG3
    _CFG3 = workloads.cfg3()
    B = _CFG3.x.shape[0]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_dense_task, range(B), chunksize=4)
    dt = time.perf_counter() - t0
    mc = max(len(r[4]) for r in res)
    errors = np.full((B, mc), np.nan)
    duals = np.full((B, mc), np.nan)
    for k, r in enumerate(res):
        errors[k, :len(r[4])] = r[4]
        duals[k, :len(r[5])] = r[5]
    its = np.array([r[0] for r in res])
    print(f"cfg3: {B} problems in {dt:.0f}s, iterations {np.unique(its, return_counts=True)}")
    save("full_cfg3_all", eps=_CFG3.eps, iterations=its, converged=np.array([r[1] for r in res]),
         f=np.stack([r[2] for r in res]).astype(np.float32),
         g=np.stack([r[3] for r in res]).astype(np.float32),
         f_absmax=np.array([np.max(np.abs(r[2])) for r in res]),
         g_absmax=np.array([np.max(np.abs(r[3])) for r in res]),
         n_checks=np.array([len(r[4]) for r in res]), errors=errors, dual_trace=duals,
         transport=np.array([r[6] for r in res]), dual=np.array([r[7] for r in res]),
         seconds=np.array(dt), procs=np.array(procs))


def conv_check(k, path, procs, chunk_blocks):
    """The reference's check pass (sinkhorn.py:181-186) in float64 at the
    potentials a GPU solve converged with (tools/dump_potentials.py)."""
    wl = workloads.make(k)
    n, m = wl.shape
    z = np.load(path)
    f = z["f"].astype(np.float64)
    g = z["g"].astype(np.float64)
    eps = float(wl.eps)
    prob_a = osink._as_weights(wl.a, n, "a")
    prob_b = osink._as_weights(wl.b, m, "b")
    t0 = time.perf_counter()
    with _pool(wl.x, wl.y, procs) as pool:
        geom = PooledPointCloud(pool, n, m, chunk_blocks)
        row = np.exp(geom.apply_lse_kernel(f, g, eps, axis="rows") / eps)
    err = float(np.abs(row - prob_a).sum())
    dual = osink._dual_objective(f, g, prob_a, prob_b, eps, row.sum())
    dt = time.perf_counter() - t0
    print(f"cfg{k}: f64 check at the GPU potentials (iteration {int(z['iterations'])}): "
          f"err={err:.6e} (GPU {float(z['gpu_error']):.6e}) threshold={wl.threshold} {dt:.0f}s")
    save(f"conv_cfg{k}", eps=np.array(eps), iterations=z["iterations"], f=z["f"], g=z["g"],
         gpu_error=z["gpu_error"], gpu_dual=z["gpu_dual"], gpu_converged=z["gpu_converged"],
         ref_error=np.array(err), ref_dual=np.array(dual), threshold=np.array(wl.threshold),
         seconds=np.array(dt))


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)", flush=True)


# (config, max_iters, chunk blocks) of the fixed-iteration fixtures
FULL = {"cfg2": (2, 2, 4), "cfg5": (5, 2, 4), "cfg4": (4, 1, 8),
        "cfg2tol": (2, None, 4), "cfg5tol": (5, None, 4), "cfg4tol": (4, None, 8)}


def main():
    procs = int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 8))
    which = sys.argv[1:]
    for w in which:
        if w in FULL:
            k, iters, cb = FULL[w]
            full_solve(k, iters, procs, cb)
        elif w == "cfg3":
            cfg3_all(procs)
        elif w.startswith("conv"):
            _, k, path = w.split(":", 2)
            conv_check(int(k), path, procs, 8)
        else:
            raise SystemExit(f"unknown fixture {w!r}")
    with open(os.path.join(HERE, "MANIFEST_fullsize.json"), "w") as fh:
        json.dump({"reference": "/root/reference/pkg (otkit 0.1.0)", "numpy": np.__version__,
                   "generated_by": "tests/golden/make_fullsize_golden.py",
                   "procs": procs, "when": time.strftime("%Y-%m-%d")}, fh, indent=1)


if __name__ == "__main__":
    main()
