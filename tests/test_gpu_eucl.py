"""cost_fn="eucl" on the GPU (reference geometry.py:274-275).

C = sqrt(max(|x|^2 + |y|^2 - 2<x,y>, 0)), exact-zero diagonal for identical
sets.  Every kernel that forms a cost carries the square root (OTK_COST_EUCL):
the tcgen05 epilogue, the FP32 low-d / tiled kernels, the persistent small
solve, reg_ot_cost, transport_matrix, the materialised cost and the
barycenter's support cost.  Checked against fixtures the reference wrote
(tests/golden/eucl.npz) and the float64 oracle.
"""

import threading

import numpy as np
import pytest

import oracle
from conftest import load_golden

pytestmark = pytest.mark.gpu

POT_TOL = 1e-4      # north star, potentials (relative, inf-norm)
COST_TOL = 1e-5     # north star, regularised OT cost
LSE_TOL = 3e-5      # single half-step vs the reference (sqrt adds ~1 ulp / cell)


@pytest.fixture(scope="module")
def otk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as m
    return m


def cases():
    fx = load_golden("eucl")
    names = sorted({k.split("__")[0] for k in fx})
    return [(nm, {k.split("__")[1]: v for k, v in fx.items() if k.startswith(nm + "__")})
            for nm in names]


def rel_inf(got, want, floor=1e-30):
    """||got - want||_inf / max(||want||_inf, floor).  For identical point sets
    the reference's g stays ~1e-12 (f carries the whole potential), so its
    errors are measured against eps (the potentials' natural scale) instead."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    return float(np.max(np.abs(got[fin] - want[fin])) / max(np.max(np.abs(want[fin])), floor))


def _geom(otk, c, impl):
    from paper_2201_12324_b200 import _native as N
    x = c["x"]
    y = x if bool(c["same"]) else c["y"]
    geom = otk.PointCloudGeometry(x, y, "eucl")
    geom.impl_flags = {"simt": N.OTK_IMPL_SIMT, "tc": N.OTK_IMPL_TC, "auto": 0}[impl]
    return geom


@pytest.mark.parametrize("impl", ["auto", "simt"])
def test_apply_lse_kernel_matches_reference(otk, impl):
    for name, c in cases():
        geom = _geom(otk, c, impl)
        eps = float(c["eps"])
        for axis in ("rows", "cols"):
            err = rel_inf(geom.apply_lse_kernel(c["f"], c["g"], eps, axis), c[axis])
            assert err <= LSE_TOL, (name, impl, axis, err)


@pytest.mark.parametrize("impl", ["auto", "simt", "nopersist"])
def test_solve_matches_reference(otk, impl):
    """Full solves: same iterations / converged flag, potentials and costs within tolerance.
    auto = the one-kernel small solve (any d at these sizes); nopersist = the tcgen05 loop;
    simt = FP32 loop."""
    from paper_2201_12324_b200 import _native as N
    for name, c in cases():
        geom = _geom(otk, c, "simt" if impl == "simt" else "auto")
        if impl == "nopersist":
            geom.impl_flags |= N.OTK_IMPL_NOPERSIST
        prob = otk.LinearProblem(geom)
        out = otk.solve_sinkhorn(prob, float(c["solve_eps"]), threshold=1e-3, max_iters=2000,
                                 impl="simt" if impl == "simt" else "auto")
        assert out.iterations == int(c["iterations"]), (name, impl)
        assert out.converged == bool(c["converged"])
        eps = float(c["solve_eps"])
        assert rel_inf(out.f, c["sol_f"], eps) <= POT_TOL, (name, impl)
        assert rel_inf(out.g, c["sol_g"], eps) <= POT_TOL, (name, impl)
        cost = otk.reg_ot_cost(out, prob)
        assert abs(cost.transport_cost - float(c["transport"])) <= COST_TOL * abs(float(c["transport"]))
        assert abs(cost.dual_objective - float(c["dual"])) <= COST_TOL * abs(float(c["dual"]))


def test_cost_matrix_transport_and_mean(otk):
    for name, c in cases():
        geom = _geom(otk, c, "auto")
        x = c["x"].astype(np.float64)
        y = x if bool(c["same"]) else c["y"].astype(np.float64)
        ref = oracle.PointCloudOracle(x, y, cost_fn="eucl")
        C = ref.cost_matrix()
        np.testing.assert_allclose(geom.cost_matrix(), C, atol=2e-5 * max(1.0, C.max()))
        if bool(c["same"]):
            assert np.all(np.diag(geom.cost_matrix()) == 0.0)
        assert geom.mean_cost() == pytest.approx(float(c["mean_cost"]), rel=1e-5)
        out = otk.solve_sinkhorn(otk.LinearProblem(geom), float(c["solve_eps"]),
                                 threshold=1e-3, max_iters=2000)
        P = otk.transport_matrix(out, otk.LinearProblem(geom)).matrix
        Pref = np.exp((c["sol_f"][:, None] + c["sol_g"][None, :] - C) / float(c["solve_eps"]))
        assert np.max(np.abs(P - Pref)) <= 1e-3 * np.max(Pref)


def test_grad_points_refuses_eucl(otk):
    c = cases()[0][1]
    geom = _geom(otk, c, "auto")
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, float(c["solve_eps"]))
    with pytest.raises(ValueError):
        otk.grad_points(out, prob)


def test_identical_sets_tc_diagonal(otk):
    """tcgen05 eucl epilogue forces C_ii = 0 (the split products leave ~1e-6 |x|^2,
    whose square root would be ~1e-3 |x|): rows LSE vs the oracle at a small eps."""
    from paper_2201_12324_b200 import _native as N
    rng = np.random.default_rng(3)
    x = rng.standard_normal((300, 64)).astype(np.float32)
    geom = otk.PointCloudGeometry(x, x, "eucl")
    geom.impl_flags = N.OTK_IMPL_TC
    ref = oracle.PointCloudOracle(x.astype(np.float64), x.astype(np.float64), cost_fn="eucl")
    eps = 0.01 * ref.mean_cost()
    g = np.zeros(300)
    got = geom.apply_lse_kernel(np.zeros(300), g, eps, "rows")
    want = ref.apply_lse_kernel(np.zeros(300), g, eps, "rows")
    assert np.max(np.abs(got - want)) <= 1e-4 * eps


def test_sharded_thread_ranks(otk):
    """Row-sharded loop with cost_fn="eucl" (2 thread ranks on one GPU) vs the oracle."""
    from paper_2201_12324_b200.sharded import ThreadComm, reg_ot_cost_sharded, shard_rows
    from paper_2201_12324_b200.sharded import solve_sinkhorn_sharded
    rng = np.random.default_rng(11)
    x = rng.standard_normal((500, 5)).astype(np.float32)
    y = (rng.standard_normal((420, 5)) + 0.5).astype(np.float32)
    ref_geom = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64), cost_fn="eucl")
    eps = 0.05 * ref_geom.mean_cost()
    ref = oracle.sinkhorn(ref_geom, None, None, eps, threshold=1e-300, max_iters=20)
    comms = ThreadComm.group(2)
    outs, costs, errs = [None, None], [None, None], []
    a, b = np.full(500, 1 / 500), np.full(420, 1 / 420)

    def run(r):
        try:
            o = solve_sinkhorn_sharded(x, y, eps, comm=comms[r], threshold=1e-300, max_iters=20,
                                       inner_iters=20, gather_f=True, cost_fn="eucl")
            lo, hi = shard_rows(500, 2, r)
            costs[r] = reg_ot_cost_sharded(o, x[lo:hi], y, a[lo:hi], b, comm=comms[r],
                                           cost_fn="eucl")
            outs[r] = o
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            comms[r].shared.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    if errs:
        raise errs[0]
    assert rel_inf(outs[0].f, ref["f"]) <= POT_TOL and rel_inf(outs[0].g, ref["g"]) <= POT_TOL
    tc, _ = oracle.reg_ot_cost(ref_geom, ref["f"], ref["g"], a, b, eps)
    assert abs(costs[0].transport_cost - tc) <= COST_TOL * abs(tc)


def test_barycenter_eucl_support(otk):
    from oracle.barycenter_oracle import solve_barycenter as ref_solve
    rng = np.random.default_rng(12)
    x = rng.standard_normal((120, 2)).astype(np.float32).astype(np.float64)
    h = rng.random((3, 120))
    h /= h.sum(axis=1, keepdims=True)
    rgeom = oracle.PointCloudOracle(x, x, cost_fn="eucl")
    eps = 0.05 * rgeom.mean_cost()
    out = otk.solve_barycenter(otk.BarycenterProblem(otk.PointCloudGeometry(x, x, "eucl"), h), eps)
    p, conv, iters, _ = ref_solve(rgeom, h, None, eps)
    assert out.converged and conv
    assert float(np.abs(out.barycenter - p).sum()) <= 1e-4


@pytest.mark.gpu
def test_device_constructor_flags_and_mean_cost_sample(otk):
    """PointCloudGeometry built from CUDA tensors: the constructor's finiteness
    and same-points tests run as one native launch (otk_points_flags,
    geometry.py:247-261) and the eps estimate's seeded 1000-pair sample as
    another (otk_mean_cost_pairs, geometry.py:294-312) -- same answers as the
    host path, which follows the reference line by line."""
    import torch
    rng = np.random.default_rng(21)
    x = rng.standard_normal((300, 5)).astype(np.float32)
    y = (rng.standard_normal((300, 5)) + 0.3).astype(np.float32)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    assert otk.PointCloudGeometry(xd, xd.clone())._same_points          # equal values, different objects
    assert not otk.PointCloudGeometry(xd, yd)._same_points
    y1 = x.copy()
    y1[299, 4] += 1e-3                                                   # one differing coordinate, the last
    assert not otk.PointCloudGeometry(xd, torch.from_numpy(y1).cuda())._same_points
    assert not otk.PointCloudGeometry(xd, yd[:200])._same_points        # shapes differ: never compared
    for bad, which in ((np.nan, "x"), (np.inf, "y"), (-np.inf, "y")):
        xb, yb = x.copy(), y.copy()
        (xb if which == "x" else yb)[17, 2] = bad
        with pytest.raises(ValueError, match="non-finite"):
            otk.PointCloudGeometry(torch.from_numpy(xb).cuda(), torch.from_numpy(yb).cuda())
    for cost_fn in ("sqeucl", "eucl", "cosine"):
        for same in (False, True):
            host = otk.PointCloudGeometry(x, x if same else y, cost_fn=cost_fn)
            dev = otk.PointCloudGeometry(xd, xd if same else yd, cost_fn=cost_fn)
            ref = oracle.PointCloudOracle(x.astype(np.float64), (x if same else y).astype(np.float64),
                                          cost_fn=cost_fn)
            assert dev.mean_cost() == pytest.approx(host.mean_cost(), rel=1e-6)
            assert dev.mean_cost() == pytest.approx(ref.mean_cost(), rel=1e-5)
