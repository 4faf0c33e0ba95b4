"""Pin the CPU oracle against fixtures produced by the reference itself.

The fixtures in tests/golden were written by tests/golden/make_golden.py,
which imports the unmodified reference (`otkit`).  If the oracle matches
them, it is a faithful checker for the CUDA path.  (CPU only.)
"""

import json

import numpy as np
import pytest
from scipy.special import logsumexp as scipy_lse

import oracle
from conftest import load_golden
from paper_2201_12324_b200 import workloads


def test_logsumexp_restatement_matches_scipy():
    rng = np.random.default_rng(0)
    z = rng.standard_normal((7, 50)) * 30
    z[0, :] = -np.inf
    z[1, 3] = -np.inf
    z[2, :] = 1e6
    for axis in (0, 1):
        np.testing.assert_allclose(oracle.logsumexp(z, axis), scipy_lse(z, axis=axis),
                                   rtol=1e-15, atol=0)
    assert oracle.logsumexp(np.full((1, 4), -np.inf), 1)[0] == -np.inf


def test_lse_pointcloud_cases_match_reference():
    fx = load_golden("lse_pointcloud")
    keys = sorted({k.split("__")[0] for k in fx})
    assert len(keys) == 12
    for key in keys:
        c = {k.split("__")[1]: v for k, v in fx.items() if k.startswith(key + "__")}
        x = c["x"].astype(np.float64)
        y = x if bool(c["same"]) else c["y"].astype(np.float64)
        geom = oracle.PointCloudOracle(x, y, block_size=37)
        eps = float(c["eps"])
        np.testing.assert_allclose(geom.apply_lse_kernel(c["f"], c["g"], eps, "rows"), c["rows"],
                                   rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(geom.apply_lse_kernel(c["f"], c["g"], eps, "cols"), c["cols"],
                                   rtol=1e-12, atol=1e-12)


def test_known_answers():
    ka = load_golden("known_answers")
    np.testing.assert_allclose(ka["log2"], np.log(2.0), rtol=1e-14)
    np.testing.assert_allclose(ka["minus_inf"], 0.0, atol=1e-14)
    geom = oracle.PointCloudOracle(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    out = oracle.sinkhorn(geom, None, None, float(ka["two_point_eps"]))
    np.testing.assert_allclose(out["f"], ka["two_point_f"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(out["g"], ka["two_point_g"], rtol=1e-12, atol=1e-12)
    assert out["iterations"] == int(ka["two_point_iters"])
    cost = oracle.reg_ot_cost(geom, out["f"], out["g"], np.full(2, .5), np.full(2, .5), out["eps"])
    np.testing.assert_allclose(cost, ka["two_point_cost"], rtol=1e-10)
    assert abs(cost[0] - 0.625) <= 1e-2
    xs = np.array([[0.0], [1.0], [2.0], [3.0]])
    geom = oracle.PointCloudOracle(xs, xs)
    assert geom.same_points
    out = oracle.sinkhorn(geom, None, None, float(ka["self_eps"]))
    np.testing.assert_allclose(out["f"], ka["self_f"], rtol=1e-12, atol=1e-12)
    sched = oracle.EpsilonScheduleOracle(float(ka["sched_target"]), 100.0, 0.5)
    geom = oracle.PointCloudOracle(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    out = oracle.sinkhorn(geom, None, None, sched, threshold=1e-6, max_iters=10_000)
    assert out["iterations"] == int(ka["sched_iters"])
    np.testing.assert_allclose(out["errors"], ka["sched_errors"], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("name", ["cfg1_small", "cfg2_small", "cfg4_small", "cfg5_small",
                                  "short_nonconv", "nonuniform_small"])
def test_solves_match_reference(name):
    fx = load_golden("solve_" + name)
    wl = getattr(workloads, str(fx["gen"]))(**json.loads(str(fx["kw"])))
    assert float(fx["eps"]) == wl.eps
    geom = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    out = oracle.sinkhorn(geom, wl.a, wl.b, wl.eps, threshold=float(fx["threshold"]),
                          max_iters=int(fx["max_iters"]))
    assert out["iterations"] == int(fx["iterations"])
    assert out["converged"] == bool(fx["converged"])
    np.testing.assert_allclose(out["f"], fx["f"], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(out["g"], fx["g"], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(out["errors"], fx["errors"], rtol=1e-7, atol=1e-13)
    np.testing.assert_allclose(out["dual_trace"], fx["dual_trace"], rtol=1e-11)
    a = oracle.as_weights(wl.a, wl.shape[0])
    b = oracle.as_weights(wl.b, wl.shape[1])
    cost = oracle.reg_ot_cost(geom, out["f"], out["g"], a, b, out["eps"])
    np.testing.assert_allclose(cost, [fx["transport"], fx["dual"]], rtol=1e-11)


def test_dense_cfg3_problems_match_reference():
    fx = load_golden("dense_cfg3")
    wl = workloads.cfg3(batch=2)
    for k in range(2):
        cost = oracle.PointCloudOracle(wl.x[k].astype(np.float64),
                                       wl.y[k].astype(np.float64)).cost_matrix()
        geom = oracle.DenseOracle(cost)
        out = oracle.sinkhorn(geom, None, None, float(wl.eps[k]), threshold=wl.threshold,
                              max_iters=wl.max_iters)
        assert out["iterations"] == int(fx[f"p{k}_iters"])
        np.testing.assert_allclose(out["f"], fx[f"p{k}_f"], rtol=1e-11, atol=1e-11)


def test_spot_cfg2_rows_subset_matches_reference():
    fx = load_golden("spot_cfg2")
    wl = workloads.cfg2()
    geom = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    rows = fx["rows"][:64]
    got = geom.rows_lse_subset(rows, fx["g"].astype(np.float64), float(fx["eps"]))
    np.testing.assert_allclose(got, fx["rows_g"][:64], rtol=1e-12)


def test_workload_eps_values_are_stable():
    # The quoted magnitudes from SURVEY.md §8d.
    assert abs(workloads.cfg1().eps - 0.339) < 0.01
    assert abs(workloads.cfg2(n=8192, m=8192).eps - 10.4) < 0.3


def barycenter_cases():
    """(name, dict) per barycenter fixture case (tests/golden/make_golden.py)."""
    fx = load_golden("barycenter")
    names = sorted({k.split("__")[0] for k in fx})
    return [(nm, {k.split("__")[1]: v for k, v in fx.items() if k.startswith(nm + "__")})
            for nm in names]


def test_barycenter_oracle_matches_reference():
    from oracle.barycenter_oracle import solve_barycenter
    cases = barycenter_cases()
    assert len(cases) == 7
    for name, c in cases:
        if c["cost"].size:
            geom = oracle.DenseOracle(c["cost"])
        else:
            geom = oracle.PointCloudOracle(c["support"], c["support"])
        p, conv, iters, _ = solve_barycenter(geom, c["hists"], c["weights"], float(c["eps"]),
                                             float(c["threshold"]), int(c["max_iters"]))
        assert iters == int(c["iterations"]), name
        assert conv == bool(c["converged"]), name
        np.testing.assert_allclose(p, c["barycenter"], rtol=1e-9, atol=1e-13, err_msg=name)


def test_barycenter_oracle_validation():
    from oracle.barycenter_oracle import solve_barycenter
    geom = oracle.PointCloudOracle(np.linspace(0, 1, 5)[:, None], np.linspace(0, 1, 5)[:, None])
    good = np.full((2, 5), 0.2)
    for hists, w in ((np.full((2, 5), 0.3), None), (good, np.array([0.5, 0.6])),
                     (np.full((2, 4), 0.25), None)):
        with pytest.raises(ValueError):
            solve_barycenter(geom, hists, w, 0.1)
    with pytest.raises(ValueError):
        solve_barycenter(oracle.DenseOracle(np.zeros((2, 3))), good, None, 0.1)
    with pytest.raises(ValueError):
        solve_barycenter(geom, good, None, -1.0)


def eucl_cases():
    fx = load_golden("eucl")
    names = sorted({k.split("__")[0] for k in fx})
    return [(nm, {k.split("__")[1]: v for k, v in fx.items() if k.startswith(nm + "__")})
            for nm in names]


def test_eucl_oracle_matches_reference():
    """cost_fn="eucl" (geometry.py:274-275): oracle LSE, solve and mean cost vs the reference."""
    cases = eucl_cases()
    assert len(cases) == 6
    for name, c in cases:
        x = c["x"].astype(np.float64)
        y = x if bool(c["same"]) else c["y"].astype(np.float64)
        geom = oracle.PointCloudOracle(x, y, cost_fn="eucl")
        eps = float(c["eps"])
        np.testing.assert_allclose(geom.apply_lse_kernel(c["f"], c["g"], eps, "rows"), c["rows"],
                                   rtol=1e-12, atol=1e-12, err_msg=name)
        np.testing.assert_allclose(geom.apply_lse_kernel(c["f"], c["g"], eps, "cols"), c["cols"],
                                   rtol=1e-12, atol=1e-12, err_msg=name)
        assert geom.mean_cost() == pytest.approx(float(c["mean_cost"]), rel=1e-12)
        ref = oracle.sinkhorn(geom, None, None, float(c["solve_eps"]), threshold=1e-3,
                              max_iters=2000)
        assert ref["iterations"] == int(c["iterations"]), name
        np.testing.assert_allclose(ref["f"], c["sol_f"], rtol=1e-9, atol=1e-12, err_msg=name)
