"""tcgen05 (split-fp16) half-step kernel vs the FP32 kernel and the float64 oracle."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def otk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as m
    from paper_2201_12324_b200 import _native
    _native.lib()
    return m


def _half_steps(otk, x, y, f, g, eps, impl):
    from paper_2201_12324_b200 import _native as N
    geom = otk.PointCloudGeometry(x, y)
    geom.impl_flags = N.OTK_IMPL_TC if impl == "tc" else N.OTK_IMPL_SIMT
    return (geom.apply_lse_kernel(f, g, eps, "rows"), geom.apply_lse_kernel(f, g, eps, "cols"))


@pytest.mark.parametrize("n,m,d", [(128, 256, 64), (300, 517, 64), (1000, 700, 128),
                                   (257, 1031, 96), (640, 384, 256), (200, 300, 1024),
                                   (4096, 4096, 64), (1, 1, 40)])
def test_tc_matches_oracle(otk, n, m, d):
    rng = np.random.default_rng(n * 7 + m + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.3 * rng.standard_normal((m, d)) + 0.2).astype(np.float32)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = 0.05 * float(np.mean([np.sum((x[i] - y[j]) ** 2) for i, j in
                                zip(rng.integers(0, n, 200), rng.integers(0, m, 200))]))
    f = (rng.standard_normal(n) * eps).astype(np.float32).astype(np.float64)
    g = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
    ref_r = geom64.apply_lse_kernel(f, g, eps, "rows")
    ref_c = geom64.apply_lse_kernel(f, g, eps, "cols")
    tr, tcol = _half_steps(otk, x, y, f, g, eps, "tc")
    scale_r = np.max(np.abs(ref_r))
    scale_c = np.max(np.abs(ref_c))
    assert np.max(np.abs(tr - ref_r)) / scale_r <= 1e-5
    assert np.max(np.abs(tcol - ref_c)) / scale_c <= 1e-5


def test_tc_unit_sphere_small_eps(otk):
    """cfg5-like regime (unit vectors, eps = 0.01 * mean)."""
    rng = np.random.default_rng(5)
    n, m, d = 512, 640, 1024
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = rng.standard_normal((m, d))
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    x, y = x.astype(np.float32), y.astype(np.float32)
    eps = 0.02
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    f = np.zeros(n)
    g = (rng.standard_normal(m) * 0.01).astype(np.float32).astype(np.float64)
    ref = geom64.apply_lse_kernel(f, g, eps, "rows")
    got, _ = _half_steps(otk, x, y, f, g, eps, "tc")
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-5


def test_tc_minus_inf_bias_columns(otk):
    rng = np.random.default_rng(1)
    n, m, d = 300, 600, 64
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = rng.standard_normal((m, d)).astype(np.float32)
    g = rng.standard_normal(m) * 5
    g[rng.random(m) < 0.5] = -np.inf
    f = np.zeros(n)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    ref = geom64.apply_lse_kernel(f, g, 10.0, "rows")
    got, _ = _half_steps(otk, x, y, f, g, 10.0, "tc")
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-5
    g[:] = -np.inf
    got, _ = _half_steps(otk, x, y, f, g, 10.0, "tc")
    assert np.all(got == -np.inf)


def test_tc_deterministic(otk):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((3000, 64)).astype(np.float32)
    y = rng.standard_normal((2500, 64)).astype(np.float32)
    f = np.zeros(3000)
    g = rng.standard_normal(2500)
    a1, b1 = _half_steps(otk, x, y, f, g, 7.0, "tc")
    a2, b2 = _half_steps(otk, x, y, f, g, 7.0, "tc")
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(b1, b2)


@pytest.mark.parametrize("d,eps_scale", [(64, 0.05), (130, 0.01), (16, 0.02)])
def test_tc_identical_point_sets(otk, d, eps_scale):
    """x is y on the tcgen05 path: the same-points instantiation forces the exact
    zero diagonal of geometry.py:278-292 like the FP32 kernels; potentials and
    cost must match the float64 oracle at the parity tolerance."""
    rng = np.random.default_rng(d)
    x = rng.standard_normal((300, d)).astype(np.float32)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), x.astype(np.float64))
    eps = eps_scale * float(geom64.cost_matrix().mean())
    ref = oracle.sinkhorn(geom64, None, None, eps, threshold=1e-300, max_iters=30)
    prob = otk.LinearProblem(otk.PointCloudGeometry(x, x))
    out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=30, impl="tc")
    # the symmetric fixed point can put all of the pair's scale in one potential
    # (the other ~0): measure both against the pair's scale, no eps floor
    scale = max(np.max(np.abs(ref["f"])), np.max(np.abs(ref["g"])))
    for got, want in ((out.f, ref["f"]), (out.g, ref["g"])):
        assert np.max(np.abs(got - want)) <= 1e-4 * scale
    assert np.all(np.diag(prob.geom.cost_matrix()) == 0.0)
    a = np.full(300, 1 / 300)
    tc, _ = oracle.reg_ot_cost(geom64, ref["f"], ref["g"], a, a, eps)
    # small eps: off-diagonal mass underflows and the cost itself is ~1e-24
    assert abs(otk.reg_ot_cost(out, prob).transport_cost - tc) <= 1e-5 * abs(tc) + 1e-12 * eps


@pytest.mark.parametrize("n,m,d", [(128, 256, 64), (300, 517, 40), (1000, 700, 128), (129, 1031, 96)])
def test_cta_pair_kernel_is_bitwise_the_single_cta_kernel(otk, n, m, d, monkeypatch):
    """The cta_group::2 (2-SM MMA) variant computes every row with the same
    MMA sequence as the 1-CTA kernel: outputs must be bitwise identical,
    including odd row-tile counts (the pair's second CTA past the last row)."""
    from paper_2201_12324_b200 import _native as N
    rng = np.random.default_rng(n + m + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (1.3 * rng.standard_normal((m, d)) + 0.2).astype(np.float32)
    eps = 0.15 * d
    f = (rng.standard_normal(n) * eps).astype(np.float32).astype(np.float64)
    g = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
    outs = []
    for pair in ("0", "1"):
        monkeypatch.setenv("OTK_TC_PAIR", pair)
        geom = otk.PointCloudGeometry(x, y)
        geom.impl_flags = N.OTK_IMPL_TC
        outs.append((geom.apply_lse_kernel(f, g, eps, "rows"), geom.apply_lse_kernel(f, g, eps, "cols")))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("seed", range(12))
def test_tc_random_shapes_every_d(otk, seed):
    """The tcgen05 kernel serves every d: random n, m (odd, tiny, tile-crossing)
    and d (1 .. 300, across the V1 / pair / V2 / V4 layouts) against the float64
    oracle, both axes, including -inf potentials (zero weights)."""
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([1, 2, 3, 5, 17, 63, 64, 65, 100, 127, 128, 129, 200, 300]))
    n = int(rng.integers(1, 700))
    m = int(rng.integers(1, 700))
    x = (rng.standard_normal((n, d)) * rng.uniform(0.2, 3.0)).astype(np.float32)
    y = (rng.standard_normal((m, d)) * rng.uniform(0.2, 3.0) + rng.uniform(-1, 1)).astype(np.float32)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = float(rng.uniform(0.02, 0.2)) * float(np.mean(geom64.cost_matrix()) + 1e-3)
    f = (rng.standard_normal(n) * eps).astype(np.float32).astype(np.float64)
    g = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
    if n > 3:
        f[rng.integers(0, n)] = -np.inf
    if m > 3:
        g[rng.integers(0, m)] = -np.inf
    ref_r = geom64.apply_lse_kernel(f, g, eps, "rows")
    ref_c = geom64.apply_lse_kernel(f, g, eps, "cols")
    tr, tcol = _half_steps(otk, x, y, f, g, eps, "tc")
    for got, ref in ((tr, ref_r), (tcol, ref_c)):
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(got), fin)
        scale = max(np.max(np.abs(ref[fin])), eps)
        assert np.max(np.abs(got[fin] - ref[fin])) / scale <= 1e-5, (n, m, d)
