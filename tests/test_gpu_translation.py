"""Translated point clouds: a common offset must not cost accuracy (needs a B200).

The reference forms _cost_block (geometry.py:268-273) in float64, where a
common offset of both clouds is harmless.  The device kernels form
|x|^2 + |y|^2 - 2<x,y> in float32 (or split fp16), so they run on clouds
shifted by one common centre (geometry.centered_points: the coordinate-wise
median of y).
These cases put both clouds at offsets of 10, 100 and 1000 per coordinate and
hold every device path to the north-star tolerances against the float64
oracle on the same float32 inputs.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

POT_TOL = 1e-4
COST_TOL = 1e-5


@pytest.fixture(scope="module")
def otk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as m
    from paper_2201_12324_b200 import _native
    _native.lib()
    return m


def rel_inf(got, want):
    return float(np.max(np.abs(np.asarray(got) - want)) / np.max(np.abs(want)))


def _clouds(d, n, m, offset, seed):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((n, d)) + offset).astype(np.float32)
    y = (1.3 * rng.standard_normal((m, d)) + offset + 0.4).astype(np.float32)
    return x, y


@pytest.mark.parametrize("offset", [10.0, 100.0, 1000.0])
@pytest.mark.parametrize("d,n,m,impl", [(3, 700, 600, "auto"), (3, 700, 600, "simt"),
                                        (3, 2500, 2300, "nopersist"), (64, 600, 500, "auto"),
                                        (64, 600, 500, "simt"), (1024, 256, 300, "auto")])
def test_offset_clouds_match_oracle(otk, d, n, m, impl, offset):
    from paper_2201_12324_b200 import _native as N
    x, y = _clouds(d, n, m, offset, seed=d + n)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    C = geom64.cost_matrix()
    eps = 0.05 * float(C.mean())
    iters = 20
    ref = oracle.sinkhorn(geom64, None, None, eps, threshold=1e-300, max_iters=iters)
    geom = otk.PointCloudGeometry(x, y)
    geom.impl_flags = {"auto": 0, "simt": N.OTK_IMPL_SIMT, "nopersist": N.OTK_IMPL_NOPERSIST}[impl]
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=iters)
    ef, eg = rel_inf(out.f, ref["f"]), rel_inf(out.g, ref["g"])
    assert ef <= POT_TOL and eg <= POT_TOL, (ef, eg)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    tc, dual = oracle.reg_ot_cost(geom64, ref["f"], ref["g"], a, b, eps)
    cost = otk.reg_ot_cost(out, prob)
    assert abs(cost.transport_cost / tc - 1.0) <= COST_TOL
    assert abs(cost.dual_objective / dual - 1.0) <= COST_TOL
    # one half-step through the plugin seam (apply_lse_kernel, geometry.py:336-354)
    rows = geom.apply_lse_kernel(np.zeros(n), ref["g"], eps, "rows")
    want = geom64.apply_lse_kernel(np.zeros(n), ref["g"], eps, "rows")
    assert rel_inf(rows, want) <= 2e-5


@pytest.mark.parametrize("offset", [100.0, 1000.0])
def test_offset_grad_points_and_cost_matrix(otk, offset):
    """grad_points (2(r x - P y), sinkhorn.py:244-246) and cost_matrix are
    translation-invariant too."""
    x, y = _clouds(16, 300, 260, offset, seed=5)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    C = geom64.cost_matrix()
    geom = otk.PointCloudGeometry(x, y)
    np.testing.assert_allclose(geom.cost_matrix(), C, rtol=2e-5, atol=2e-5 * C.mean())
    eps = 0.05 * float(C.mean())
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, eps, threshold=1e-4, max_iters=3000)
    assert out.converged
    plan = np.exp((out.f[:, None] + out.g[None, :] - C) / out.eps)
    want = 2.0 * (plan.sum(axis=1)[:, None] * x.astype(np.float64) - plan @ y.astype(np.float64))
    got = otk.grad_points(out, prob)
    assert np.max(np.abs(got - want)) <= 1e-4 * np.max(np.abs(want))


def test_identical_offset_sets_exact_zero_diagonal(otk):
    """x is y at an offset: the exact-zero diagonal (geometry.py:259-261,
    278-292) on the tcgen05 path as well.  The symmetric problem's fixed point
    puts everything in f (the reference's g is ~1e-14), so both potentials are
    measured against the pair's scale max(|f|, |g|) -- the scale of the
    (f + c, g - c) invariance -- with the plain 1e-4 gate, no eps floor."""
    rng = np.random.default_rng(3)
    for d in (3, 64, 200):
        x = (rng.standard_normal((300, d)) + 100.0).astype(np.float32)
        geom64 = oracle.PointCloudOracle(x.astype(np.float64), x.astype(np.float64))
        C = geom64.cost_matrix()
        eps = 0.02 * float(C.mean())
        ref = oracle.sinkhorn(geom64, None, None, eps, threshold=1e-300, max_iters=15)
        for flags in (0,):
            geom = otk.PointCloudGeometry(x, x)
            geom.impl_flags = flags
            prob = otk.LinearProblem(geom)
            out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=15)
            scale = max(np.max(np.abs(ref["f"])), np.max(np.abs(ref["g"])))
            assert np.max(np.abs(out.f - ref["f"])) <= POT_TOL * scale
            assert np.max(np.abs(out.g - ref["g"])) <= POT_TOL * scale
            assert np.all(np.diag(geom.cost_matrix()) == 0.0)
            # self-matching known answer (test_sinkhorn.py:50-58 setting): tiny transport cost
            a = np.full(300, 1 / 300)
            tc, _ = oracle.reg_ot_cost(geom64, ref["f"], ref["g"], a, a, eps)
            got = otk.reg_ot_cost(out, prob).transport_cost
            assert abs(got - tc) <= COST_TOL * max(abs(tc), 1e-3 * float(C.mean())), (got, tc)
