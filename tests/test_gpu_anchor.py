"""Anchored half-steps (otk_lse_step): the fixed-anchor tcgen05 epilogue and its
device-side repair path, against the running-max kernel and the float64 oracle.

The anchored kernel sums 2^(u_ij - anchor_i) with the anchor taken from the
row's previous result; rows whose result leaves the safe window are
recomputed by the running-max kernel inside the same call.  These tests feed
deliberately wrong anchors (far above, far below, NaN, +inf) and check that
every row comes out as the running-max result.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as otk
    from paper_2201_12324_b200 import _native as N
    N.lib()
    return otk, N, torch


def _setup(env, n, m, d, seed):
    otk, N, torch = env
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.5 * rng.standard_normal((m, d))).astype(np.float32)
    geom = otk.PointCloudGeometry(x, y)
    geom.impl_flags = N.OTK_IMPL_TC
    cx, cy = geom._clouds()
    eps = 0.05 * float(np.mean(np.sum((x[:64, None, :] - y[None, :64, :]) ** 2, axis=-1)))
    g = (rng.standard_normal(m) * 3 * eps).astype(np.float32)
    return x, y, geom, cx, cy, eps, g


def _step(env, geom, cx, cy, g, eps, anchor=None, init=False, mode=None, rep=None):
    """One rows half-step through otk_lse_step; returns the output vector."""
    otk, N, torch = env
    lib = N.lib()
    from paper_2201_12324_b200._device import stream
    n, m = cx.n, cy.n
    kappa = float(np.float32(1.4426950408889634 / eps))
    dev = cx.p.device
    gt = torch.as_tensor(g, device=dev)
    bias = torch.empty(m, dtype=torch.float32, device=dev)
    N.check(lib.otk_make_bias(N.ptr(gt), m, kappa, N.ptr(bias), None, 0, stream()))
    flags = N.OTK_CLAMP | N.OTK_IMPL_TC | (N.OTK_ANCHOR_INIT if init else 0)
    nsplit = lib.otk_lse_suggest_nsplit(n, m, cx.d, flags)
    part = torch.empty(nsplit * n, dtype=torch.float32, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    base = torch.full((n,), float(np.log(1.0 / n)), dtype=torch.float32, device=dev)
    if rep is None:
        rep = torch.empty(lib.otk_lse_step_workspace_bytes(n), dtype=torch.uint8, device=dev)
    mode = N.OTK_FIN_LOG2 if mode is None else mode
    N.check(lib.otk_lse_step(N.ptr(cx.p), N.ptr(cx.sq), N.ptr(cx.hi), N.ptr(cx.lo), N.ptr(cx.ext_a), n,
                             N.ptr(cy.p), N.ptr(cy.sq), N.ptr(cy.hi), N.ptr(cy.lo), N.ptr(cy.ext_b), m,
                             cx.d, cx.dpad, 1.0 / (cx.scale * cx.scale), N.ptr(bias), kappa, flags,
                             nsplit, N.ptr(part), N.ptr(base), mode, float(eps), kappa, N.ptr(out),
                             None, None, 0, N.ptr(anchor), N.ptr(rep), None, stream()),
            "otk_lse_step")
    torch.cuda.synchronize()
    return out.cpu().numpy(), rep


@pytest.mark.parametrize("n,m,d", [(1000, 3000, 64), (700, 1300, 128), (513, 900, 200),
                                   (300, 700, 300), (128, 256, 16)])
def test_anchor_init_and_perfect_anchor(env, n, m, d):
    otk, N, torch = env
    x, y, geom, cx, cy, eps, g = _setup(env, n, m, d, n + d)
    plain, _ = _step(env, geom, cx, cy, g, eps)
    anchor = torch.full((n,), float("nan"), device=cx.p.device)
    init, _ = _step(env, geom, cx, cy, g, eps, anchor=anchor, init=True)
    assert np.array_equal(init, plain)  # INIT runs the running-max kernel
    assert np.array_equal(anchor.cpu().numpy(), plain)
    anch, rep = _step(env, geom, cx, cy, g, eps, anchor=anchor)
    tol = 2e-6 * np.maximum(1.0, np.abs(plain))
    assert np.all(np.abs(anch - plain) <= tol), np.max(np.abs(anch - plain))
    assert int(rep[:4].view(torch.int32).item()) == 0  # nothing repaired
    # the oracle agrees (log2 units: L_i = log2 sum_j 2^(kappa (g_j - C_ij)))
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    ref = geom64.apply_lse_kernel(np.zeros(n), g.astype(np.float64), eps, "rows") / (eps * np.log(2.0))
    assert np.max(np.abs(anch - ref)) <= 1e-5 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("n,m,d", [(1000, 3000, 64), (700, 1300, 128), (300, 700, 300)])
def test_anchor_repair_bad_anchors(env, n, m, d):
    """Anchors 200 above (flush), 300 below (overflow), NaN and +inf: those rows'
    tiles are recomputed by the running-max kernel -> bitwise the plain result."""
    otk, N, torch = env
    x, y, geom, cx, cy, eps, g = _setup(env, n, m, d, 3 * n + d)
    plain, _ = _step(env, geom, cx, cy, g, eps)
    a = plain.copy()
    rng = np.random.default_rng(7)
    a += rng.uniform(-3.0, 3.0, n).astype(np.float32)  # harmless offsets
    bad = {5: 200.0, 130: -300.0, 131: float("nan"), n - 1: float("inf")}
    for i, v in bad.items():
        a[i] = v if not np.isfinite(v) else a[i] + v
    anchor = torch.as_tensor(a, device=cx.p.device)
    out, rep = _step(env, geom, cx, cy, g, eps, anchor=anchor)
    flagged_tiles = sorted({i // 128 for i in bad})
    assert int(rep[:4].view(torch.int32).item()) == len(bad)
    for t in flagged_tiles:
        sl = slice(128 * t, min(n, 128 * (t + 1)))
        assert np.array_equal(out[sl], plain[sl]), t
    tol = 2e-6 * np.maximum(1.0, np.abs(plain))
    assert np.all(np.abs(out - plain) <= tol)
    assert np.array_equal(anchor.cpu().numpy(), out)  # anchors now hold this result


def test_anchor_solver_mode_matches_partial_finalize(env):
    """SOLVER mode through otk_lse_step == otk_lse_partial + otk_lse_finalize."""
    otk, N, torch = env
    n, m, d = 640, 900, 64
    x, y, geom, cx, cy, eps, g = _setup(env, n, m, d, 11)
    anchor = torch.full((n,), float("nan"), device=cx.p.device)
    f_init, _ = _step(env, geom, cx, cy, g, eps, anchor=anchor, init=True, mode=N.OTK_FIN_SOLVER)
    f_anch, _ = _step(env, geom, cx, cy, g, eps, anchor=anchor, mode=N.OTK_FIN_SOLVER)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    ref = eps * np.log(1.0 / n) - geom64.apply_lse_kernel(np.zeros(n), g.astype(np.float64), eps, "rows")
    for got in (f_init, f_anch):
        assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-5


@pytest.fixture
def anchor_always(monkeypatch):
    """The solver anchors only long half-steps by default (>= 2^27 cells); these
    tests exercise the anchored path at small sizes."""
    monkeypatch.setenv("OTK_ANCHOR_MIN_CELLS", "0")


@pytest.mark.parametrize("d", [64, 128])
def test_solver_anchored_vs_running_max(env, d, anchor_always):
    """Whole solves: anchored (default) vs running-max only -- same iterations and
    convergence, potentials within fp32 noise; far-off warm start forces repairs."""
    otk, N, torch = env
    rng = np.random.default_rng(d)
    n, m = 3000, 2500
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.5 * rng.standard_normal((m, d))).astype(np.float32)
    prob = otk.LinearProblem(otk.PointCloudGeometry(x, y))
    eps = 0.05 * float(np.mean(np.sum((x[:64, None, :] - y[None, :64, :]) ** 2, axis=-1)))
    for g_init in (None, (rng.standard_normal(m) * 400 * eps).astype(np.float32)):
        kw = dict(threshold=1e-3, max_iters=300, g_init=g_init)
        a = otk.solve_sinkhorn(prob, eps, impl="tc", **kw)
        b = otk.solve_sinkhorn(prob, eps, impl="tc-noanchor", **kw)
        assert a.iterations == b.iterations and a.converged == b.converged
        for name in ("f", "g"):
            u, v = getattr(a, name), getattr(b, name)
            assert np.max(np.abs(u - v)) / np.max(np.abs(v)) <= 2e-6, name
        assert np.allclose(a.errors, b.errors, rtol=1e-3, atol=1e-6)


def test_solver_anchored_graph_periods(env, anchor_always):
    """Long fixed-iteration solve (CUDA-graph periods replayed many times) stays
    on the running-max trajectory."""
    otk, N, torch = env
    rng = np.random.default_rng(3)
    n, m, d = 2048, 2048, 64
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.5 * rng.standard_normal((m, d))).astype(np.float32)
    prob = otk.LinearProblem(otk.PointCloudGeometry(x, y))
    eps = 0.05 * float(np.mean(np.sum((x[:64, None, :] - y[None, :64, :]) ** 2, axis=-1)))
    kw = dict(threshold=1e-300, max_iters=120)
    a = otk.solve_sinkhorn(prob, eps, impl="tc", **kw)
    b = otk.solve_sinkhorn(prob, eps, impl="tc-noanchor", **kw)
    # either run may stop early at an exact fp32 fixed point (err == 0 <= 1e-300);
    # past it the potentials no longer move, so the two stay comparable.  At
    # least two graph-captured check periods ran in each.
    assert a.iterations >= 20 and b.iterations >= 20
    assert a.converged == (a.iterations < 120) and b.converged == (b.iterations < 120)
    for name in ("f", "g"):
        u, v = getattr(a, name), getattr(b, name)
        assert np.max(np.abs(u - v)) / np.max(np.abs(v)) <= 1e-5, name


def test_anchored_solver_zero_weights_and_small_eps(env, anchor_always):
    """Zero weights on both sides (-inf potentials, empty plan rows/columns) and a
    small eps (most terms far below each row's maximum) on the anchored tcgen05
    path: same trajectory as the running-max path and the float64 oracle."""
    otk, N, torch = env
    rng = np.random.default_rng(17)
    n, m, d = 700, 900, 64
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.5 * rng.standard_normal((m, d))).astype(np.float32)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.5, 1.5, m)
    a[rng.choice(n, 40, replace=False)] = 0.0
    b[rng.choice(m, 55, replace=False)] = 0.0
    a /= a.sum()
    b /= b.sum()
    mean_c = float(np.mean(np.sum((x[:64, None, :] - y[None, :64, :]) ** 2, axis=-1)))
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    for scale, its in ((0.05, 30), (0.005, 40)):
        eps = scale * mean_c
        prob = otk.LinearProblem(otk.PointCloudGeometry(x, y), a, b)
        out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=its, impl="tc")
        ref_rm = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=its, impl="tc-noanchor")
        ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-300, max_iters=its)
        assert np.array_equal(np.isneginf(out.f), a == 0) and np.array_equal(np.isneginf(out.g), b == 0)
        for name in ("f", "g"):
            got, rm, want = getattr(out, name), getattr(ref_rm, name), ref[name]
            fin = np.isfinite(want)
            scale_ = np.max(np.abs(want[fin]))
            assert np.max(np.abs(got[fin] - rm[fin])) / scale_ <= 2e-6, (scale, name)
            assert np.max(np.abs(got[fin] - want[fin])) / scale_ <= 1e-4, (scale, name)
