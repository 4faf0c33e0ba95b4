"""Fixed-support barycenters (reference otkit/barycenter.py).

CPU: problem validation mirrors barycenter.py:39-64 / 96-106 (no device).
GPU: the one-launch CUDA solve (csrc/bary.cu) against the fixtures the
reference wrote (tests/golden/barycenter.npz: same iterations and converged
flag, barycenter within fp32 tolerance), against the float64 oracle on
random supports, and the reference test-suite's invariants
(tests/test_barycenter.py of the reference: single histogram, identical
histograms, Dirac midpoints and weight interpolation, probability vector,
support permutation, zero entries).
"""

import numpy as np
import pytest

import paper_2201_12324_b200 as otk
from conftest import load_golden
from paper_2201_12324_b200 import _native as N

# fp32 kernels: |p_gpu - p_ref|_1 after identical iteration counts.
BARY_L1_TOL = 2e-5


def line_geometry(n):
    pts = np.linspace(0.0, 1.0, n)
    return otk.PointCloudGeometry(pts[:, None], pts[:, None]), pts


def dirac(n, i):
    h = np.zeros(n)
    h[i] = 1.0
    return h


def cases():
    fx = load_golden("barycenter")
    names = sorted({k.split("__")[0] for k in fx})
    return [(nm, {k.split("__")[1]: v for k, v in fx.items() if k.startswith(nm + "__")})
            for nm in names]


# ---------------------------------------------------------------- CPU
def test_problem_validation():
    geom, _ = line_geometry(5)
    good = np.full((2, 5), 0.2)
    with pytest.raises(ValueError):
        otk.BarycenterProblem(geom, np.full((2, 5), 0.3))
    with pytest.raises(ValueError):
        otk.BarycenterProblem(geom, good, np.array([0.5, 0.6]))
    with pytest.raises(ValueError):
        otk.BarycenterProblem(geom, np.full((2, 4), 0.25))
    with pytest.raises(ValueError):
        otk.BarycenterProblem(otk.DenseGeometry(np.zeros((2, 3))), good)
    with pytest.raises(ValueError):
        otk.BarycenterProblem(geom, good, np.array([0.5, np.nan]))
    with pytest.raises(ValueError):
        otk.BarycenterProblem(geom, -good)
    with pytest.raises(ValueError):
        otk.solve_barycenter(otk.BarycenterProblem(geom, good), -1.0)
    with pytest.raises(ValueError):
        otk.solve_barycenter(otk.BarycenterProblem(geom, good), 0.1, max_iters=0)
    with pytest.raises(ValueError):
        otk.solve_barycenter(otk.BarycenterProblem(geom, good), 0.1, threshold=0.0)
    bp = otk.BarycenterProblem(geom, good[0])           # 1-D histogram -> (1, N)
    assert bp.histograms.shape == (1, 5) and bp.weights.tolist() == [1.0]


def test_barycenter_symbols_exported():
    lib = N.lib()
    for name in ("otk_solve_barycenter", "otk_barycenter_part_len", "otk_barycenter_pad",
                 "otk_barycenter_ld"):
        assert hasattr(lib, name)


# ---------------------------------------------------------------- GPU
def _geom_of(c):
    if c["cost"].size:
        return otk.DenseGeometry(c["cost"])
    return otk.PointCloudGeometry(c["support"], c["support"])


@pytest.mark.gpu
def test_matches_reference_fixtures():
    for name, c in cases():
        bp = otk.BarycenterProblem(_geom_of(c), c["hists"], c["weights"])
        out = otk.solve_barycenter(bp, float(c["eps"]), threshold=float(c["threshold"]),
                                   max_iters=int(c["max_iters"]))
        assert out.iterations == int(c["iterations"]), name
        assert out.converged == bool(c["converged"]), name
        l1 = float(np.abs(out.barycenter - c["barycenter"]).sum())
        assert l1 <= BARY_L1_TOL, (name, l1)
        assert out.eps == float(c["eps"])
        assert len(out.errors) == out.iterations


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k,eps_rel,dense", [(96, 2, 3, 0.05, False), (257, 3, 5, 0.03, False),
                                                 (512, 8, 2, 0.02, False), (300, 0, 4, 0.05, True)])
def test_matches_oracle_random(n, d, k, eps_rel, dense):
    import oracle
    from oracle.barycenter_oracle import solve_barycenter as ref_solve
    rng = np.random.default_rng(n + k)
    if dense:
        C = rng.uniform(0, 1, (n, n)).astype(np.float32).astype(np.float64)
        geom, rgeom = otk.DenseGeometry(C), oracle.DenseOracle(C)
    else:
        x = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
        geom, rgeom = otk.PointCloudGeometry(x, x), oracle.PointCloudOracle(x, x)
    h = rng.random((k, n)) ** 3
    h /= h.sum(axis=1, keepdims=True)
    w = rng.random(k)
    w /= w.sum()
    eps = eps_rel * rgeom.mean_cost()
    out = otk.solve_barycenter(otk.BarycenterProblem(geom, h, w), eps, threshold=1e-4)
    p, conv, iters, _ = ref_solve(rgeom, h, w, eps, 1e-4, 1000)
    assert out.converged and conv
    assert abs(out.iterations - iters) <= max(2, iters // 50), (out.iterations, iters)
    assert float(np.abs(out.barycenter - p).sum()) <= 1e-4


@pytest.mark.gpu
def test_fixed_iterations_match_oracle():
    """Fixed iteration count (threshold unreachable): same trajectory as the oracle."""
    import oracle
    from oracle.barycenter_oracle import solve_barycenter as ref_solve
    rng = np.random.default_rng(5)
    x = rng.standard_normal((203, 4)).astype(np.float32).astype(np.float64)
    h = rng.random((3, 203))
    h /= h.sum(axis=1, keepdims=True)
    rgeom = oracle.PointCloudOracle(x, x)
    eps = 0.05 * rgeom.mean_cost()
    for iters in (1, 7, 40):
        out = otk.solve_barycenter(otk.BarycenterProblem(otk.PointCloudGeometry(x, x), h), eps,
                                   threshold=1e-300, max_iters=iters)
        p, conv, t, _ = ref_solve(rgeom, h, None, eps, 1e-300, iters)
        assert out.iterations == t == iters and not out.converged and not conv
        assert float(np.abs(out.barycenter - p).sum()) <= BARY_L1_TOL, iters


@pytest.mark.gpu
def test_single_histogram_is_its_own_barycenter():
    geom, _ = line_geometry(21)
    h = np.random.default_rng(0).random(21)
    h /= h.sum()
    out = otk.solve_barycenter(otk.BarycenterProblem(geom, h[None, :]), 1e-5 * geom.mean_cost())
    assert out.converged
    assert np.abs(out.barycenter - h).sum() <= 1e-6


@pytest.mark.gpu
def test_identical_histograms_are_a_fixed_point():
    geom, _ = line_geometry(21)
    h = np.random.default_rng(1).random(21)
    h /= h.sum()
    bp = otk.BarycenterProblem(geom, np.stack([h, h]), np.array([0.3, 0.7]))
    out = otk.solve_barycenter(bp, 1e-5 * geom.mean_cost())
    assert np.abs(out.barycenter - h).sum() <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("weights,target", [(None, 0.5), ((0.3, 0.7), 0.3 * 0.25 + 0.7 * 0.75)])
def test_dirac_interpolation(weights, target):
    geom, pts = line_geometry(101)
    hists = np.stack([dirac(101, 25), dirac(101, 75)])
    w = None if weights is None else np.array(weights)
    out = otk.solve_barycenter(otk.BarycenterProblem(geom, hists, w), 1e-3 * geom.mean_cost())
    assert int(np.argmax(out.barycenter)) == int(np.argmin(np.abs(pts - target)))


@pytest.mark.gpu
def test_output_is_a_probability_vector():
    geom, _ = line_geometry(31)
    hists = np.random.default_rng(2).random((3, 31))
    hists /= hists.sum(axis=1, keepdims=True)
    out = otk.solve_barycenter(otk.BarycenterProblem(geom, hists), 1e-2 * geom.mean_cost())
    assert np.all(out.barycenter >= 0)
    assert abs(out.barycenter.sum() - 1.0) <= 1e-10
    assert out.iterations >= 1
    assert out.eps == 1e-2 * geom.mean_cost()


@pytest.mark.gpu
def test_permuting_the_support_permutes_the_barycenter():
    rng = np.random.default_rng(3)
    pts = np.sort(rng.random(9))
    geom = otk.PointCloudGeometry(pts[:, None], pts[:, None])
    hists = rng.random((2, 9))
    hists /= hists.sum(axis=1, keepdims=True)
    eps = 1e-2 * geom.mean_cost()
    base = otk.solve_barycenter(otk.BarycenterProblem(geom, hists), eps)
    perm = rng.permutation(9)
    C = np.asarray(geom.cost_matrix(), dtype=np.float64)
    permuted = otk.solve_barycenter(
        otk.BarycenterProblem(otk.DenseGeometry(np.asarray(C)[np.ix_(perm, perm)]), hists[:, perm]), eps)
    np.testing.assert_allclose(base.barycenter[perm], permuted.barycenter, atol=1e-6)


@pytest.mark.gpu
def test_zero_entries_and_determinism():
    geom, _ = line_geometry(11)
    hists = np.stack([dirac(11, 0), dirac(11, 10)])
    bp = otk.BarycenterProblem(geom, hists)
    out = otk.solve_barycenter(bp, 1e-3 * geom.mean_cost())
    assert abs(out.barycenter.sum() - 1.0) <= 1e-10
    again = otk.solve_barycenter(bp, 1e-3 * geom.mean_cost())
    assert np.array_equal(out.barycenter, again.barycenter)


@pytest.mark.gpu
def test_cosine_support_and_launch_count():
    """Cosine support (kernel points x/|x|/sqrt2) vs the oracle on the explicit cosine cost."""
    import oracle
    from oracle.barycenter_oracle import solve_barycenter as ref_solve
    rng = np.random.default_rng(9)
    x = rng.standard_normal((128, 6)).astype(np.float32).astype(np.float64)
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    C = np.maximum(1.0 - xn @ xn.T, 0.0)
    np.fill_diagonal(C, 0.0)
    h = rng.random((2, 128))
    h /= h.sum(axis=1, keepdims=True)
    eps = 0.05 * C.mean()
    out = otk.solve_barycenter(otk.BarycenterProblem(otk.PointCloudGeometry(x, x, "cosine"), h), eps)
    p, conv, iters, _ = ref_solve(oracle.DenseOracle(C), h, None, eps, 1e-4, 1000)
    assert out.converged and conv
    assert float(np.abs(out.barycenter - p).sum()) <= 1e-4


@pytest.mark.gpu
def test_eps_below_fp32_range_raises():
    """log2(e)/eps must be a finite fp32 (documented limit of the device kernels)."""
    geom, _ = line_geometry(11)
    hists = np.stack([dirac(11, 0), dirac(11, 10)])
    with pytest.raises(ValueError):
        otk.solve_barycenter(otk.BarycenterProblem(geom, hists), 1e-45)
