"""Generate golden fixtures by running the REFERENCE (`otkit`) itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

It imports the unmodified reference package and records its outputs on
seeded inputs into ``tests/golden/*.npz``.  The fixtures travel with the repo
(the reference does not exist on the GPU box) and pin both the CPU oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_parity.py).

Inputs are either stored in the fixture (small cases) or regenerated on the
box from ``paper_2201_12324_b200.workloads`` (full-size configs), whose numpy
draws are deterministic.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import otkit  # noqa: E402  (reference, from PYTHONPATH)
import otkit.geometry as ogeo  # noqa: E402
import scipy  # noqa: E402

from paper_2201_12324_b200 import workloads  # noqa: E402

OUT = HERE


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def solve_ref(x, y, a, b, eps, threshold, max_iters, inner_iters=10, same=False):
    x64 = np.asarray(x, np.float64)
    y64 = x64 if same else np.asarray(y, np.float64)
    geom = otkit.PointCloudGeometry(x64, y64)
    prob = otkit.LinearProblem(geom, a, b)
    out = otkit.solve_sinkhorn(prob, eps, threshold=threshold, max_iters=max_iters,
                               inner_iters=inner_iters)
    old = ogeo.DEFAULT_DENSE_CAP
    ogeo.DEFAULT_DENSE_CAP = max(old, geom.shape[0] * geom.shape[1])
    try:
        cost = otkit.reg_ot_cost(out, prob)
    finally:
        ogeo.DEFAULT_DENSE_CAP = old
    return out, cost


def lse_cases():
    """PointCloud apply_lse_kernel on random small clouds (rows & cols), incl. -inf
    potentials and identical point sets."""
    rng = np.random.default_rng(12324)
    cases = {}
    for k in range(12):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(1, 300))
        d = int(rng.integers(1, 70))
        same = k % 4 == 3
        if same:
            m = n
        x = rng.standard_normal((n, d)).astype(np.float32)
        y = x if same else (rng.standard_normal((m, d)) + 0.3).astype(np.float32)
        x64 = x.astype(np.float64)
        y64 = x64 if same else y.astype(np.float64)
        geom = otkit.PointCloudGeometry(x64, y64, block_size=int(rng.integers(1, 300)))
        eps = float(0.3 * geom.mean_cost() + 1e-3)
        f = (rng.standard_normal(n) * eps * 2).astype(np.float32).astype(np.float64)
        g = (rng.standard_normal(m) * eps * 2).astype(np.float32).astype(np.float64)
        if k % 3 == 1:
            g[rng.random(m) < 0.3] = -np.inf
            f[rng.random(n) < 0.3] = -np.inf
        rows = geom.apply_lse_kernel(f, g, eps, "rows")
        cols = geom.apply_lse_kernel(f, g, eps, "cols")
        cases[f"c{k}"] = dict(x=x, y=y, same=same, eps=eps, f=f, g=g, rows=rows, cols=cols)
    flat = {}
    for key, c in cases.items():
        for kk, v in c.items():
            flat[f"{key}__{kk}"] = np.asarray(v)
    save("lse_pointcloud", **flat)


def known_answers():
    """Pinned values from the reference's own tests, recomputed by the reference."""
    res = {}
    # test_geometry.py:154-157: all-zero cost -> log 2
    res["log2"] = otkit.DenseGeometry(np.zeros((2, 2))).apply_lse_kernel(
        np.zeros(2), np.zeros(2), 1.0, "rows")
    # test_geometry.py:181-184: -inf potential
    res["minus_inf"] = otkit.DenseGeometry(np.zeros((2, 2))).apply_lse_kernel(
        np.zeros(2), np.array([0.0, -np.inf]), 1.0, "rows")
    # test_sinkhorn.py:41-47 two-point problem through the PointCloud path
    geom = otkit.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    prob = otkit.LinearProblem(geom)
    eps2 = 1e-3 * geom.mean_cost()
    out = otkit.solve_sinkhorn(prob, eps2)
    res["two_point_eps"] = np.array(eps2)
    res["two_point_f"] = out.f
    res["two_point_g"] = out.g
    res["two_point_iters"] = np.array(out.iterations)
    res["two_point_cost"] = np.array(otkit.reg_ot_cost(out, prob))
    res["two_point_plan"] = otkit.transport_matrix(out, prob).matrix
    # test_sinkhorn.py:50-58 self-matching (identical point sets)
    xs = np.array([[0.0], [1.0], [2.0], [3.0]])
    geom = otkit.PointCloudGeometry(xs, xs)
    prob = otkit.LinearProblem(geom)
    eps_s = 1e-3 * geom.mean_cost()
    out = otkit.solve_sinkhorn(prob, eps_s)
    res["self_eps"] = np.array(eps_s)
    res["self_f"] = out.f
    res["self_g"] = out.g
    res["self_cost"] = np.array(otkit.reg_ot_cost(out, prob))
    res["self_iters"] = np.array(out.iterations)
    # singleton point cloud x=[0], y=[3] (test_sinkhorn.py:202-206 setting)
    geom = otkit.PointCloudGeometry(np.array([[0.0]]), np.array([[3.0]]))
    prob = otkit.LinearProblem(geom)
    out = otkit.solve_sinkhorn(prob, 1.0)
    res["single_f"] = out.f
    res["single_g"] = out.g
    res["single_cost"] = np.array(otkit.reg_ot_cost(out, prob))
    # large-eps independent coupling (test_sinkhorn.py:61-66)
    geom = otkit.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.0], [1.0]]))
    prob = otkit.LinearProblem(geom)
    out = otkit.solve_sinkhorn(prob, 1e3 * geom.mean_cost())
    res["bigeps_plan"] = otkit.transport_matrix(out, prob).matrix
    res["bigeps_eps"] = np.array(1e3 * geom.mean_cost())
    # zero-weight column through the PointCloud path (test_sinkhorn.py:235-241 setting)
    geom = otkit.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.2], [0.9]]))
    prob = otkit.LinearProblem(geom, None, np.array([1.0, 0.0]))
    out = otkit.solve_sinkhorn(prob, 0.5)
    res["zerow_f"] = out.f
    res["zerow_g"] = out.g
    res["zerow_plan"] = otkit.transport_matrix(out, prob).matrix
    # epsilon schedule (test_sinkhorn.py:129-136 setting)
    geom = otkit.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    prob = otkit.LinearProblem(geom)
    target = 1e-3 * geom.mean_cost()
    out = otkit.solve_sinkhorn(prob, otkit.EpsilonSchedule(target, init_scale=100.0, decay=0.5),
                               threshold=1e-6, max_iters=10_000)
    res["sched_target"] = np.array(target)
    res["sched_f"] = out.f
    res["sched_g"] = out.g
    res["sched_iters"] = np.array(out.iterations)
    res["sched_errors"] = out.errors
    res["sched_cost"] = np.array(otkit.reg_ot_cost(out, prob))
    save("known_answers", **res)


def solve_cases():
    """Full solves at sizes the reference finishes in seconds (plus cfg1 at full size)."""
    specs = [
        # name, generator, kwargs, threshold override, max_iters override
        ("cfg1_small", workloads.cfg1, dict(n=256, m=192), None, None),
        ("cfg1_full", workloads.cfg1, dict(), None, None),
        ("cfg2_small", workloads.cfg2, dict(n=1024, m=768), None, None),
        ("cfg4_small", workloads.cfg4, dict(n=1024, m=512), None, None),
        ("cfg5_small", workloads.cfg5, dict(n=512, m=512), None, None),
        ("short_nonconv", workloads.cfg2, dict(n=512, m=512), 1e-12, 7),
        ("nonuniform_small", workloads.cfg4, dict(n=300, m=200, d=5), 1e-6, 5000),
    ]
    for name, gen, kw, thr, mi in specs:
        wl = gen(**kw)
        t0 = time.perf_counter()
        out, cost = solve_ref(wl.x, wl.y, wl.a, wl.b, wl.eps,
                              wl.threshold if thr is None else thr,
                              wl.max_iters if mi is None else mi)
        dt = time.perf_counter() - t0
        print(f"{name}: iters={out.iterations} converged={out.converged} {dt:.1f}s")
        save(f"solve_{name}", gen=np.array(gen.__name__), kw=np.array(json.dumps(kw)),
             threshold=np.array(wl.threshold if thr is None else thr),
             max_iters=np.array(wl.max_iters if mi is None else mi),
             eps=np.array(wl.eps), f=out.f, g=out.g, errors=out.errors,
             dual_trace=out.dual_trace, iterations=np.array(out.iterations),
             converged=np.array(out.converged), transport=np.array(cost.transport_cost),
             dual=np.array(cost.dual_objective), seconds=np.array(dt))


def fixed_iter_cases():
    """Fixed-iteration runs (threshold 1e-300 never met): bit-level f/g comparison
    target of BASELINE.json configs[0], plus reduced versions of cfg2/cfg4/cfg5."""
    specs = [
        ("cfg1_fixed200", workloads.cfg1, dict(), 200),
        ("cfg2_fixed20", workloads.cfg2, dict(n=2048, m=2048), 20),
        ("cfg4_fixed20", workloads.cfg4, dict(n=2048, m=1024), 20),
        ("cfg5_fixed30", workloads.cfg5, dict(n=1024, m=1024), 30),
    ]
    for name, gen, kw, iters in specs:
        wl = gen(**kw)
        t0 = time.perf_counter()
        out, cost = solve_ref(wl.x, wl.y, wl.a, wl.b, wl.eps, 1e-300, iters)
        dt = time.perf_counter() - t0
        print(f"{name}: {dt:.1f}s err={out.errors[-1]:.3e}")
        save(f"fixed_{name}", gen=np.array(gen.__name__), kw=np.array(json.dumps(kw)),
             iters=np.array(iters), eps=np.array(wl.eps), f=out.f, g=out.g,
             errors=out.errors, dual_trace=out.dual_trace,
             transport=np.array(cost.transport_cost), dual=np.array(cost.dual_objective),
             seconds=np.array(dt))


def dense_cases():
    """DenseGeometry (materialised) solves on the first problems of cfg3."""
    wl = workloads.cfg3(batch=6)
    res = {}
    for k in range(6):
        x64 = wl.x[k].astype(np.float64)
        y64 = wl.y[k].astype(np.float64)
        cost = otkit.PointCloudGeometry(x64, y64).cost_matrix(max_entries=512 * 512)
        geom = otkit.DenseGeometry(cost)
        prob = otkit.LinearProblem(geom)
        out = otkit.solve_sinkhorn(prob, float(wl.eps[k]), threshold=wl.threshold,
                                   max_iters=wl.max_iters)
        rc = otkit.reg_ot_cost(out, prob)
        res[f"p{k}_f"] = out.f
        res[f"p{k}_g"] = out.g
        res[f"p{k}_iters"] = np.array(out.iterations)
        res[f"p{k}_errors"] = out.errors
        res[f"p{k}_cost"] = np.array(rc)
        print(f"dense p{k}: iters={out.iterations}")
    save("dense_cfg3", **res)


def spot_checks():
    """Exact half-step spot checks at FULL BASELINE sizes.

    rows: eps*LSE_j((g_j - C_ij)/eps) on 256 seeded rows for g = 0 (the
    solver's first f half-step) and for a seeded g; cols: the same over i for
    256 seeded columns and a seeded f.  Inputs regenerate from workloads.py.
    """
    for k, gen in ((2, workloads.cfg2), (4, workloads.cfg4), (5, workloads.cfg5)):
        wl = gen()
        n, m = wl.shape
        rng = np.random.default_rng(777 + k)
        rows = np.sort(rng.choice(n, 256, replace=False))
        cols = np.sort(rng.choice(m, 256, replace=False))
        gpot = (rng.standard_normal(m) * 2.0 * wl.eps).astype(np.float32).astype(np.float64)
        fpot = (rng.standard_normal(n) * 2.0 * wl.eps).astype(np.float32).astype(np.float64)
        x64 = wl.x.astype(np.float64)
        y64 = wl.y.astype(np.float64)
        t0 = time.perf_counter()
        sub = otkit.PointCloudGeometry(x64[rows], y64)
        rows_g0 = sub.apply_lse_kernel(np.zeros(256), np.zeros(m), wl.eps, "rows")
        rows_g = sub.apply_lse_kernel(np.zeros(256), gpot, wl.eps, "rows")
        del sub
        subc = otkit.PointCloudGeometry(x64, y64[cols])
        cols_f = subc.apply_lse_kernel(fpot, np.zeros(256), wl.eps, "cols")
        del subc
        print(f"spot cfg{k}: {time.perf_counter() - t0:.1f}s")
        save(f"spot_cfg{k}", eps=np.array(wl.eps), rows=rows, cols=cols, g=gpot.astype(np.float32),
             f=fpot.astype(np.float32), rows_g0=rows_g0, rows_g=rows_g, cols_f=cols_f)


def eucl_cases():
    """cost_fn="eucl" (geometry.py:274-275): apply_lse_kernel rows/cols and full
    solves by the reference, incl. identical point sets and -inf potentials."""
    rng = np.random.default_rng(2201)
    res = {}
    for k, (n, m, d, same) in enumerate([(97, 130, 2, False), (200, 200, 3, True),
                                         (150, 90, 16, False), (128, 128, 64, True),
                                         (96, 140, 100, False), (64, 70, 300, False)]):
        x = rng.standard_normal((n, d)).astype(np.float32)
        y = x if same else (rng.standard_normal((m, d)) + 0.4).astype(np.float32)
        x64 = x.astype(np.float64)
        y64 = x64 if same else y.astype(np.float64)
        geom = otkit.PointCloudGeometry(x64, y64, "eucl")
        eps = float(0.2 * geom.mean_cost())
        f = (rng.standard_normal(n) * eps).astype(np.float32).astype(np.float64)
        g = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
        if k % 2 == 1:
            g[rng.random(m) < 0.2] = -np.inf
        rows = geom.apply_lse_kernel(f, g, eps, "rows")
        cols = geom.apply_lse_kernel(f, g, eps, "cols")
        solve_eps = float(0.05 * geom.mean_cost())
        prob = otkit.LinearProblem(geom)
        out = otkit.solve_sinkhorn(prob, solve_eps, threshold=1e-3, max_iters=2000)
        old = ogeo.DEFAULT_DENSE_CAP
        ogeo.DEFAULT_DENSE_CAP = max(old, n * m)
        try:
            cost = otkit.reg_ot_cost(out, prob)
        finally:
            ogeo.DEFAULT_DENSE_CAP = old
        for key, v in dict(x=x, y=y, same=same, eps=eps, f=f, g=g, rows=rows, cols=cols,
                           solve_eps=solve_eps, sol_f=out.f, sol_g=out.g,
                           iterations=out.iterations, converged=out.converged,
                           errors=out.errors, transport=cost.transport_cost,
                           dual=cost.dual_objective, mean_cost=geom.mean_cost()).items():
            res[f"e{k}__{key}"] = np.asarray(v)
        print(f"eucl e{k}: n={n} m={m} d={d} same={same} iters={out.iterations}")
    save("eucl", **res)


def barycenter_cases():
    """Fixed-support barycenters (otkit/barycenter.py:73-133), SURVEY.md §8f row 4.

    Supports are fp32-representable (the GPU sees the same values); each case
    stores its inputs and the reference's barycenter, log p, iterations and
    converged flag.  The dense case uses a non-symmetric explicit cost.
    """
    res = {}

    def line(n):
        return np.linspace(0.0, 1.0, n).astype(np.float32).astype(np.float64)[:, None]

    def dirac(n, i):
        h = np.zeros(n)
        h[i] = 1.0
        return h

    def rand_hists(rng, k, n, zero_frac=0.0):
        h = rng.random((k, n))
        if zero_frac:
            h[rng.random((k, n)) < zero_frac] = 0.0
        return h / h.sum(axis=1, keepdims=True)

    rng = np.random.default_rng(4242)
    cases = []
    pts = line(21)
    cases.append(("single", pts, None, rand_hists(np.random.default_rng(0), 1, 21), None, 1e-5, 1e-4, 1000))
    pts = line(101)
    cases.append(("diracs", pts, None, np.stack([dirac(101, 25), dirac(101, 75)]),
                  np.array([0.3, 0.7]), 1e-3, 1e-4, 1000))
    cases.append(("zeros", line(11), None, np.stack([dirac(11, 0), dirac(11, 10)]), None, 1e-3,
                  1e-4, 1000))
    pts = rng.standard_normal((64, 2)).astype(np.float32).astype(np.float64)
    cases.append(("cloud2d", pts, None, rand_hists(rng, 3, 64), None, 0.05, 1e-4, 1000))
    pts = rng.standard_normal((200, 3)).astype(np.float32).astype(np.float64)
    w = rng.random(4)
    cases.append(("cloud3d_zeros", pts, None, rand_hists(rng, 4, 200, 0.2), w / w.sum(), 0.02,
                  1e-4, 1000))
    pts = rng.standard_normal((130, 5)).astype(np.float32).astype(np.float64)
    cases.append(("short", pts, None, rand_hists(rng, 2, 130), None, 0.01, 1e-6, 3))
    cost = rng.uniform(0.0, 1.0, (50, 50)).astype(np.float32).astype(np.float64)
    cases.append(("dense", None, cost, rand_hists(rng, 2, 50), np.array([0.6, 0.4]), 0.05, 1e-4,
                  1000))
    for name, support, cost, hists, weights, eps_rel, threshold, max_iters in cases:
        if cost is None:
            geom = otkit.PointCloudGeometry(support, support)
        else:
            geom = otkit.DenseGeometry(cost)
        eps = eps_rel * geom.mean_cost()
        bp = otkit.BarycenterProblem(geom, hists, weights)
        out = otkit.solve_barycenter(bp, eps, threshold=threshold, max_iters=max_iters)
        log_p = np.log(out.barycenter)  # normalised p; the stored target
        res[f"{name}__support"] = support if support is not None else np.zeros((0, 1))
        res[f"{name}__cost"] = cost if cost is not None else np.zeros((0, 0))
        res[f"{name}__hists"] = hists
        res[f"{name}__weights"] = bp.weights
        res[f"{name}__eps"] = np.array(eps)
        res[f"{name}__threshold"] = np.array(threshold)
        res[f"{name}__max_iters"] = np.array(max_iters)
        res[f"{name}__barycenter"] = out.barycenter
        res[f"{name}__log_p"] = log_p
        res[f"{name}__iterations"] = np.array(out.iterations)
        res[f"{name}__converged"] = np.array(out.converged)
        print(f"barycenter {name}: iters={out.iterations} converged={out.converged}")
    save("barycenter", **res)


def main():
    which = sys.argv[1:] or ["lse", "known", "solve", "fixed", "dense", "spot", "bary", "eucl"]
    meta = dict(reference="/root/reference/pkg (otkit 0.1.0)", numpy=np.__version__,
                scipy=scipy.__version__, python=platform.python_version(),
                generated_by="tests/golden/make_golden.py", when=time.strftime("%Y-%m-%d"))
    if "lse" in which:
        lse_cases()
    if "known" in which:
        known_answers()
    if "solve" in which:
        solve_cases()
    if "fixed" in which:
        fixed_iter_cases()
    if "dense" in which:
        dense_cases()
    if "spot" in which:
        spot_checks()
    if "bary" in which:
        barycenter_cases()
    if "eucl" in which:
        eucl_cases()
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
