"""CUDA path vs the oracle / reference golden fixtures (needs a B200).

Tolerances (BASELINE.json north_star, float32 device arithmetic):
  potentials f, g: ||delta||_inf / ||ref||_inf <= 1e-4
  regularised OT cost (transport, dual): relative <= 1e-5
  iteration count and converged flag: identical to the reference.
"""

import json

import numpy as np
import pytest

import oracle
from conftest import load_golden
from paper_2201_12324_b200 import workloads

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
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin), "finite pattern differs"
    assert np.array_equal(got[~fin], want[~fin])
    if not fin.any():
        return 0.0
    return float(np.max(np.abs(got[fin] - want[fin])) / max(np.max(np.abs(want[fin])), 1e-30))


# ------------------------------------------------------------------ kernels
@pytest.mark.parametrize("impl", ["simt", "auto"])
def test_apply_lse_kernel_matches_reference_cases(otk, impl):
    fx = load_golden("lse_pointcloud")
    keys = sorted({k.split("__")[0] for k in fx})
    for key in keys:
        c = {k.split("__")[1]: v for k, v in fx.items() if k.startswith(key + "__")}
        x = c["x"]
        y = x if bool(c["same"]) else c["y"]
        geom = otk.PointCloudGeometry(x, y, block_size=37)
        if impl == "simt":
            from paper_2201_12324_b200 import _native
            geom.impl_flags = _native.OTK_IMPL_SIMT
        eps = float(c["eps"])
        for axis in ("rows", "cols"):
            got = geom.apply_lse_kernel(c["f"], c["g"], eps, axis)
            err = rel_inf(got, c[axis])
            assert err <= 2e-5, f"{key} {axis}: {err:.2e}"


def test_lse_kernel_known_answers(otk):
    ka = load_golden("known_answers")
    geom = otk.DenseGeometry(np.zeros((2, 2)))
    np.testing.assert_allclose(geom.apply_lse_kernel(np.zeros(2), np.zeros(2), 1.0, "rows"),
                               ka["log2"], rtol=1e-6)
    out = geom.apply_lse_kernel(np.zeros(2), np.array([0.0, -np.inf]), 1.0, "rows")
    np.testing.assert_allclose(out, 0.0, atol=1e-6)
    with pytest.raises(ValueError):
        geom.apply_lse_kernel(np.array([0.0, np.nan]), np.zeros(2), 1.0, "rows")
    # huge offsets stay finite (test_geometry.py:160-168)
    rng = np.random.default_rng(4)
    dg = otk.DenseGeometry(rng.random((3, 4)))
    f = rng.standard_normal(3)
    g = rng.standard_normal(4)
    base = dg.apply_lse_kernel(f, g, 0.5, "rows")
    shifted = dg.apply_lse_kernel(f - 1e6, g, 0.5, "rows")
    assert np.all(np.isfinite(shifted))
    np.testing.assert_allclose(shifted + 1e6, base, atol=0.2)  # float32 ulp at 1e6 is 0.0625
    # point cloud: all-equal points -> log(m) offsets
    pc = otk.PointCloudGeometry(np.zeros((3, 2)), np.zeros((5, 2)))
    np.testing.assert_allclose(pc.apply_lse_kernel(np.zeros(3), np.zeros(5), 1.0, "rows"),
                               np.log(5.0), rtol=1e-6)


@pytest.mark.parametrize("k", [2, 4, 5])
def test_full_size_half_step_spot_checks(otk, k):
    """Exact reference half-steps on 256 rows / columns at the FULL config sizes."""
    fx = load_golden(f"spot_cfg{k}")
    wl = workloads.make(k)
    geom = otk.PointCloudGeometry(wl.x, wl.y)
    eps = float(fx["eps"])
    n, m = wl.shape
    rows0 = geom.apply_lse_kernel(np.zeros(n), np.zeros(m), eps, "rows")[fx["rows"]]
    assert rel_inf(rows0, fx["rows_g0"]) <= 2e-5
    rows_g = geom.apply_lse_kernel(np.zeros(n), fx["g"].astype(np.float64), eps, "rows")[fx["rows"]]
    assert rel_inf(rows_g, fx["rows_g"]) <= 2e-5
    cols_f = geom.apply_lse_kernel(fx["f"].astype(np.float64), np.zeros(m), eps, "cols")[fx["cols"]]
    assert rel_inf(cols_f, fx["cols_f"]) <= 2e-5


# ------------------------------------------------------------------ solves
def _solve_golden(otk, name, **kw):
    fx = load_golden(name)
    gen = getattr(workloads, str(fx["gen"]))
    wl = gen(**json.loads(str(fx["kw"])))
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    return fx, wl, prob


@pytest.mark.parametrize("name", ["cfg1_small", "cfg1_full", "cfg2_small", "cfg4_small",
                                  "cfg5_small", "short_nonconv", "nonuniform_small"])
@pytest.mark.parametrize("impl", ["auto", "simt", "tc"])  # auto: the one-kernel small solve at these sizes; tc: the tcgen05 loop
def test_solve_matches_reference(otk, name, impl):
    fx, wl, prob = _solve_golden(otk, "solve_" + name)
    out = otk.solve_sinkhorn(prob, float(fx["eps"]), threshold=float(fx["threshold"]),
                             max_iters=int(fx["max_iters"]), impl=impl)
    assert out.iterations == int(fx["iterations"])
    assert out.converged == bool(fx["converged"])
    assert len(out.errors) == len(fx["errors"])
    assert rel_inf(out.f, fx["f"]) <= POT_TOL
    assert rel_inf(out.g, fx["g"]) <= POT_TOL
    # the whole check trace (sinkhorn.py:183-186): marginal errors within 1e-3
    # relative plus four times the float32 floor ulp(max|f|)/eps, dual trace 1e-5
    floor = float(np.spacing(np.float32(np.max(np.abs(fx["f"][np.isfinite(fx["f"])]))))) / float(fx["eps"])
    np.testing.assert_allclose(out.errors, fx["errors"], rtol=1e-3, atol=4.0 * floor)
    np.testing.assert_allclose(out.dual_trace, fx["dual_trace"], rtol=COST_TOL,
                               atol=1e-6 * np.max(np.abs(fx["dual_trace"])))
    cost = otk.reg_ot_cost(out, prob)
    assert abs(cost.transport_cost - float(fx["transport"])) <= COST_TOL * abs(float(fx["transport"]))
    assert abs(cost.dual_objective - float(fx["dual"])) <= COST_TOL * abs(float(fx["dual"])) + 1e-6


@pytest.mark.parametrize("name", ["cfg1_fixed200", "cfg2_fixed20", "cfg4_fixed20", "cfg5_fixed30"])
def test_fixed_iteration_runs(otk, name):
    fx = load_golden("fixed_" + name)
    wl = getattr(workloads, str(fx["gen"]))(**json.loads(str(fx["kw"])))
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    out = otk.solve_sinkhorn(prob, float(fx["eps"]), threshold=1e-300, max_iters=int(fx["iters"]))
    # float32 iterates can reach an exact fixed point (f_{t+1} == f_t bitwise: marginal error
    # 0.0 <= 1e-300, so the loop stops there); every later iterate would be the same
    # potentials, so they still compare with the reference's at the full count
    if out.converged:
        assert out.errors[-1] == 0.0 and out.iterations <= int(fx["iters"])
    else:
        assert out.iterations == int(fx["iters"])
    assert rel_inf(out.f, fx["f"]) <= POT_TOL, rel_inf(out.f, fx["f"])
    assert rel_inf(out.g, fx["g"]) <= POT_TOL, rel_inf(out.g, fx["g"])
    k = len(out.dual_trace)
    np.testing.assert_allclose(out.dual_trace, fx["dual_trace"][:k], rtol=COST_TOL)
    cost = otk.reg_ot_cost(out, prob)
    assert abs(cost.transport_cost / float(fx["transport"]) - 1) <= COST_TOL
    assert abs(cost.dual_objective / float(fx["dual"]) - 1) <= COST_TOL


def test_bitwise_determinism(otk):
    wl = workloads.cfg2(n=1500, m=1300)
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y))
    o1 = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=25)
    o2 = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=25)
    np.testing.assert_array_equal(o1.f, o2.f)
    np.testing.assert_array_equal(o1.g, o2.g)
    np.testing.assert_array_equal(o1.errors, o2.errors)
    np.testing.assert_array_equal(o1.dual_trace, o2.dual_trace)


def test_graphs_do_not_change_results(otk):
    wl = workloads.cfg1(n=700, m=500)
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y))
    o1 = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=37, use_graphs=True)
    o2 = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=37, use_graphs=False)
    np.testing.assert_array_equal(o1.f, o2.f)
    np.testing.assert_array_equal(o1.g, o2.g)
    np.testing.assert_array_equal(o1.errors, o2.errors)


# ------------------------------------------------------------------ pinned examples
def test_pinned_point_cloud_examples(otk):
    ka = load_golden("known_answers")
    geom = otk.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, float(ka["two_point_eps"]))
    # eps = 1e-3 * mean cost: float32 potentials resolve P only to ulp(f)/eps ~ 4e-5,
    # so the slow geometric convergence crosses 1e-3 within a few checks of float64.
    assert out.converged
    assert abs(out.iterations - int(ka["two_point_iters"])) <= 0.2 * int(ka["two_point_iters"])
    cost = otk.reg_ot_cost(out, prob)
    assert abs(cost.transport_cost - 0.625) <= 1e-2
    plan = otk.transport_matrix(out, prob).matrix
    assert plan[0, 1] + plan[1, 0] <= 1e-3
    # self-matching
    xs = np.array([[0.0], [1.0], [2.0], [3.0]])
    geom = otk.PointCloudGeometry(xs, xs)
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, float(ka["self_eps"]))
    assert otk.reg_ot_cost(out, prob).transport_cost <= 1e-6
    plan = otk.transport_matrix(out, prob).matrix
    np.testing.assert_array_equal(plan.argmax(axis=1), np.arange(4))
    np.testing.assert_allclose(plan, np.eye(4) / 4.0, atol=1e-6)
    # singleton: cost 9, P = [[1]]
    geom = otk.PointCloudGeometry(np.array([[0.0]]), np.array([[3.0]]))
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, 1.0)
    np.testing.assert_allclose(otk.transport_matrix(out, prob).matrix, [[1.0]], atol=1e-6)
    np.testing.assert_allclose(otk.reg_ot_cost(out, prob), ka["single_cost"], rtol=1e-6)
    # large eps -> independent coupling
    geom = otk.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.0], [1.0]]))
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, float(ka["bigeps_eps"]))
    np.testing.assert_allclose(otk.transport_matrix(out, prob).matrix, ka["bigeps_plan"], atol=1e-6)
    # zero-weight column empties the plan column
    geom = otk.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.2], [0.9]]))
    prob = otk.LinearProblem(geom, None, np.array([1.0, 0.0]))
    out = otk.solve_sinkhorn(prob, 0.5)
    plan = otk.transport_matrix(out, prob).matrix
    np.testing.assert_allclose(plan[:, 1], 0.0, atol=1e-12)
    np.testing.assert_allclose(plan, ka["zerow_plan"], atol=1e-6)
    assert out.g[1] == -np.inf
    # epsilon schedule
    geom = otk.PointCloudGeometry(np.array([[0.0], [1.0]]), np.array([[0.5], [2.0]]))
    prob = otk.LinearProblem(geom)
    sched = otk.EpsilonSchedule(float(ka["sched_target"]), init_scale=100.0, decay=0.5)
    out = otk.solve_sinkhorn(prob, sched, threshold=1e-6, max_iters=10_000)
    # reference assertions (test_sinkhorn.py:129-136); at eps = 1.4e-3 the float32
    # marginal error floor (~ulp(f)/eps ~ 1e-5) exceeds the 1e-6 threshold, so the
    # check that first passes can come one or two checks after float64's
    assert out.converged and out.eps == float(ka["sched_target"])
    assert out.iterations <= int(ka["sched_iters"]) + 2 * 10
    assert abs(otk.reg_ot_cost(out, prob).transport_cost - 0.625) <= 1e-2


def test_failure_modes(otk):
    cost = np.array([[0.0, 2.0, 3.0], [2.0, 0.0, 3.0]])
    prob = otk.LinearProblem(otk.DenseGeometry(cost), None, np.array([0.5, 0.5, 0.0]))
    with pytest.raises(otk.DivergedError) as exc:
        otk.solve_sinkhorn(prob, 1e-320, inner_iters=1)
    assert exc.value.iteration >= 1
    prob = otk.LinearProblem(otk.DenseGeometry(np.ones((2, 2))))
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 0.0)
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 1.0, threshold=0.0)
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 1.0, max_iters=0)


# ------------------------------------------------------------------ dense / batched
def test_dense_geometry_solves_match_reference(otk):
    fx = load_golden("dense_cfg3")
    wl = workloads.cfg3(batch=3)
    for k in range(3):
        cost = oracle.PointCloudOracle(wl.x[k].astype(np.float64),
                                       wl.y[k].astype(np.float64)).cost_matrix()
        prob = otk.LinearProblem(otk.DenseGeometry(cost))
        out = otk.solve_sinkhorn(prob, float(wl.eps[k]), threshold=wl.threshold,
                                 max_iters=wl.max_iters)
        assert out.iterations == int(fx[f"p{k}_iters"])
        assert rel_inf(out.f, fx[f"p{k}_f"]) <= POT_TOL
        assert rel_inf(out.g, fx[f"p{k}_g"]) <= POT_TOL
        rc = otk.reg_ot_cost(out, prob)
        np.testing.assert_allclose(rc, fx[f"p{k}_cost"], rtol=COST_TOL)


@pytest.mark.parametrize("kernel", ["cluster", "cta"])
def test_batched_cfg3_matches_reference(otk, kernel, monkeypatch):
    """Both one-launch batched solvers: K3c (cost resident in a cluster's shared
    memory, the default) and K3p (one CTA per problem streaming C from HBM)."""
    monkeypatch.setenv("OTK_DENSE_KERNEL", kernel)
    fx = load_golden("dense_cfg3")
    wl = workloads.cfg3(batch=6)
    outs, costs = otk.solve_sinkhorn_batched(wl.x, wl.y, wl.eps, threshold=wl.threshold,
                                             max_iters=wl.max_iters, return_cost=True)
    for k in range(6):
        assert outs[k].iterations == int(fx[f"p{k}_iters"])
        assert outs[k].converged
        assert rel_inf(outs[k].f, fx[f"p{k}_f"]) <= POT_TOL
        assert rel_inf(outs[k].g, fx[f"p{k}_g"]) <= POT_TOL
        np.testing.assert_allclose(costs[k], fx[f"p{k}_cost"], rtol=COST_TOL)


def test_dense_reference_style_properties(otk):
    # test_sinkhorn.py:72-94 settings (float32 tolerances)
    rng = np.random.default_rng(8)
    geom = otk.DenseGeometry(rng.random((5, 4)))
    a = rng.random(5) + 0.2
    a /= a.sum()
    b = rng.random(4) + 0.2
    b /= b.sum()
    prob = otk.LinearProblem(geom, a, b)
    out = otk.solve_sinkhorn(prob, 0.05 * geom.mean_cost(), threshold=1e-5, max_iters=10_000)
    assert out.converged
    plan = otk.transport_matrix(out, prob)
    assert np.abs(plan.row_marginal() - a).sum() <= 1e-5
    assert np.abs(plan.col_marginal() - b).sum() <= 2e-5
    rng = np.random.default_rng(9)
    geom = otk.DenseGeometry(rng.random((6, 6)))
    out = otk.solve_sinkhorn(otk.LinearProblem(geom), 0.01 * geom.mean_cost(), threshold=1e-5,
                             max_iters=20_000)
    assert len(out.dual_trace) == len(out.errors)
    assert np.all(np.diff(out.dual_trace) >= -1e-6)


# ------------------------------------------------------------------ full-size properties
@pytest.mark.parametrize("k", [2])
def test_full_size_properties(otk, k):
    """At BASELINE sizes: first f half-step equals the reference spot values, the
    dual trace is nondecreasing and the marginal error drops."""
    wl = workloads.make(k)
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y))
    out = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=30)
    assert np.all(np.isfinite(out.f)) and np.all(np.isfinite(out.g))
    assert np.all(np.diff(out.dual_trace) >= -1e-6 * np.abs(out.dual_trace[:-1]))
    assert out.errors[0] <= wl.threshold  # converges at the first check (float64 does too)
    fx = load_golden(f"spot_cfg{k}")
    one = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=1)
    # f_1 = eps*log(1/n) - eps*LSE_j(-C_ij/eps)
    f1_ref = wl.eps * np.log(1.0 / wl.shape[0]) - fx["rows_g0"]
    assert rel_inf(one.f[fx["rows"]], f1_ref) <= 2e-5


def test_reference_loop_drives_the_drop_in_geometry(otk):
    """The reference's loop (its oracle restatement of _sinkhorn_iterations,
    sinkhorn.py:151-200) runs unchanged on top of our PointCloudGeometry: every
    half-step is otk_lse_partial + otk_lse_finalize."""
    for gen, kw in (("cfg1", dict(n=300, m=257)), ("cfg2", dict(n=384, m=320, d=64))):
        wl = getattr(workloads, gen)(**kw)
        ours = oracle.sinkhorn(otk.PointCloudGeometry(wl.x, wl.y), None, None, wl.eps,
                               threshold=1e-300, max_iters=20)
        ref = oracle.sinkhorn(oracle.PointCloudOracle(wl.x.astype(np.float64),
                                                      wl.y.astype(np.float64)),
                              None, None, wl.eps, threshold=1e-300, max_iters=20)
        assert ours["iterations"] == ref["iterations"]
        assert rel_inf(ours["f"], ref["f"]) <= POT_TOL
        assert rel_inf(ours["g"], ref["g"]) <= POT_TOL


@pytest.mark.parametrize("d,same,nonuniform", [(3, False, False), (1, False, True), (5, False, False),
                                               (3, True, False), (7, False, True), (8, False, False),
                                               (11, True, False), (16, False, True), (19, False, False),
                                               (33, False, True), (64, False, False), (130, False, False)])
def test_persistent_small_solve_matches_general_loop_and_oracle(otk, d, same, nonuniform):
    """The one-kernel small-problem solve (csrc/solve_small.cu) against the
    general launch-per-half-step loop (OTK_IMPL_NOPERSIST) and the oracle:
    same iterations / converged flag / check trace length, f and g within
    the float32 tolerance, bitwise-reproducible reruns."""
    from paper_2201_12324_b200 import _native as N
    rng = np.random.default_rng(100 + d)
    n, m = 700, (700 if same else 555)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = x if same else (rng.standard_normal((m, d)) + 0.4).astype(np.float32)
    a = b = None
    if nonuniform:
        a = rng.uniform(0.5, 1.5, n)
        a[7] = 0.0
        a /= a.sum()
        b = rng.uniform(0.5, 1.5, m)
        b /= b.sum()
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = 0.05 * float(np.mean(geom64.cost_matrix()))
    ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-3, max_iters=500)

    def run(flags):
        g = otk.PointCloudGeometry(x, y)
        g.impl_flags = flags
        return otk.solve_sinkhorn(otk.LinearProblem(g, a, b), eps, threshold=1e-3, max_iters=500)
    fast, fast2, gen = run(0), run(0), run(N.OTK_IMPL_NOPERSIST)
    for out in (fast, gen):
        assert out.iterations == ref["iterations"] and out.converged == ref["converged"]
        assert len(out.errors) == len(ref["errors"])
        assert rel_inf(out.f, ref["f"]) <= POT_TOL
        assert rel_inf(out.g, ref["g"]) <= POT_TOL
    assert np.array_equal(fast.f, fast2.f) and np.array_equal(fast.g, fast2.g)
    np.testing.assert_allclose(fast.errors, gen.errors, rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("d,n,m,same", [(3, 300, 257, False), (64, 200, 150, False),
                                        (130, 100, 90, False), (3, 120, 120, True)])
def test_grad_points_online_matches_reference_formula(otk, d, n, m, same):
    """grad_points computed online on the GPU vs the
    reference's materialised formula 2(r x - P y) (sinkhorn.py:244-246)
    evaluated in float64 at the same potentials."""
    rng = np.random.default_rng(d * 1000 + n)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = x if same else (rng.standard_normal((m, d)) * 1.2 + 0.3).astype(np.float32)
    geom = otk.PointCloudGeometry(x, y)
    prob = otk.LinearProblem(geom)
    C = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64)).cost_matrix()
    eps = 0.05 * float(C.mean())
    out = otk.solve_sinkhorn(prob, eps, threshold=1e-4, max_iters=3000)
    assert out.converged
    got = otk.grad_points(out, prob)
    plan = np.exp((out.f[:, None] + out.g[None, :] - C) / out.eps)
    want = 2.0 * (plan.sum(axis=1)[:, None] * x.astype(np.float64) - plan @ y.astype(np.float64))
    assert got.shape == want.shape and got.dtype == np.float64
    assert np.max(np.abs(got - want)) <= 1e-4 * np.max(np.abs(want))
    gw = otk.grad_weights(out, prob)
    assert abs(gw.mean()) < 1e-9 and np.allclose(gw, out.f - out.f.mean())


@pytest.mark.parametrize("path", ["small", "general", "tc", "dense", "batched"])
def test_warm_start_and_annealing_match_oracle(otk, path):
    """g_init warm starts and eps annealing (the inner
    solves of GW / low-rank / GMM, quadratic.py:169-177) on every device path
    against the oracle loop with the same g_init / schedule."""
    from paper_2201_12324_b200 import _native as N
    rng = np.random.default_rng(31)
    d = 64 if path == "tc" else 3
    n, m = 260, 230
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.3).astype(np.float32)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    C = geom64.cost_matrix()
    eps = 0.05 * float(C.mean())
    g0 = (rng.standard_normal(m) * eps).astype(np.float32).astype(np.float64)
    anneal = path in ("general", "dense")
    sched = otk.EpsilonSchedule(eps, init_scale=20.0, decay=0.6) if anneal else eps
    osched = oracle.EpsilonScheduleOracle(eps, 20.0, 0.6) if anneal else eps
    if path in ("dense", "batched"):
        ref = oracle.sinkhorn(oracle.DenseOracle(C.astype(np.float32).astype(np.float64)), None,
                              None, osched, threshold=1e-4, max_iters=400, g_init=g0)
    else:
        ref = oracle.sinkhorn(geom64, None, None, osched, threshold=1e-4, max_iters=400, g_init=g0)
    if path == "batched":
        outs = otk.solve_sinkhorn_batched(x[None], y[None], eps, threshold=1e-4, max_iters=400,
                                          g_init=g0[None])
        out = outs[0]
    elif path == "dense":
        out = otk.solve_sinkhorn(otk.LinearProblem(otk.DenseGeometry(C)), sched, threshold=1e-4,
                                 max_iters=400, g_init=g0)
    else:
        geom = otk.PointCloudGeometry(x, y)
        geom.impl_flags = {"small": 0, "general": N.OTK_IMPL_NOPERSIST, "tc": 0}[path]
        out = otk.solve_sinkhorn(otk.LinearProblem(geom), sched, threshold=1e-4, max_iters=400,
                                 g_init=g0)
    assert out.iterations == ref["iterations"] and out.converged == ref["converged"]
    assert rel_inf(out.f, ref["f"]) <= POT_TOL
    assert rel_inf(out.g, ref["g"]) <= POT_TOL


def _cosine_cost(x, y):
    """Reference cosine cost, geometry.py:265-267 (float64)."""
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    yn = y / np.linalg.norm(y, axis=1, keepdims=True)
    return 1.0 - xn @ yn.T


@pytest.mark.parametrize("d", [3, 64])
def test_cosine_cost_solve_matches_reference_formula(otk, d):
    """cost_fn="cosine": the sqeucl kernels on x^/sqrt2."""
    rng = np.random.default_rng(40 + d)
    x = (rng.standard_normal((220, d)) + 0.3).astype(np.float32)
    y = (rng.standard_normal((190, d)) - 0.2).astype(np.float32)
    C = _cosine_cost(x.astype(np.float64), y.astype(np.float64))
    geom = otk.PointCloudGeometry(x, y, cost_fn="cosine")
    np.testing.assert_allclose(geom.cost_matrix(), C, atol=2e-6)
    eps = 0.05 * float(C.mean())
    ref = oracle.sinkhorn(oracle.DenseOracle(C), None, None, eps, threshold=1e-300, max_iters=30)
    prob = otk.LinearProblem(geom)
    out = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=30)
    assert rel_inf(out.f, ref["f"]) <= POT_TOL and rel_inf(out.g, ref["g"]) <= POT_TOL
    a = np.full(220, 1 / 220)
    b = np.full(190, 1 / 190)
    tc, dual = oracle.reg_ot_cost(oracle.DenseOracle(C), ref["f"], ref["g"], a, b, eps)
    cost = otk.reg_ot_cost(out, prob)
    assert abs(cost.transport_cost - tc) <= COST_TOL * abs(tc)
    assert abs(geom.mean_cost() - float(np.mean(C))) < 0.1  # 1000-pair sample estimate


@pytest.mark.parametrize("cost_fn", ["sqeucl", "cosine"])
def test_apply_kernel_matches_dense_gibbs_product(otk, cost_fn):
    """Non-log apply_kernel (geometry.py:130-139, 318-334) on the GPU vs
    exp(-C/eps) @ v in float64, rows and cols, positive and signed v."""
    rng = np.random.default_rng(7)
    x = (rng.standard_normal((150, 3)) + 2.0).astype(np.float32)
    y = (rng.standard_normal((130, 3)) + 2.0).astype(np.float32)
    x64, y64 = x.astype(np.float64), y.astype(np.float64)
    C = _cosine_cost(x64, y64) if cost_fn == "cosine" else \
        oracle.PointCloudOracle(x64, y64).cost_matrix()
    geom = otk.PointCloudGeometry(x, y, cost_fn=cost_fn)
    eps = 0.5 * float(C.mean()) + 0.1
    K = np.exp(-C / eps)
    v, u = rng.random(130) + 0.1, rng.random(150) + 0.1
    np.testing.assert_allclose(geom.apply_kernel(v, eps, "rows"), K @ v, rtol=1e-5)
    np.testing.assert_allclose(geom.apply_kernel(u, eps, "cols"), K.T @ u, rtol=1e-5)
    vs = rng.standard_normal(130)
    got = geom.apply_kernel(vs, eps, "rows")
    assert np.all(np.abs(got - K @ vs) <= 1e-5 * (np.abs(K) @ np.abs(vs)))
    dense = otk.DenseGeometry(C)
    np.testing.assert_allclose(dense.apply_kernel(v, eps, "rows"), K @ v, rtol=1e-5)
    # known answers (test_geometry.py:61-68)
    np.testing.assert_allclose(otk.DenseGeometry(np.array([[0.0]])).apply_kernel(
        np.array([1.0]), 1.0, "rows"), [1.0], rtol=1e-6)
    np.testing.assert_allclose(otk.DenseGeometry(np.zeros((2, 2))).apply_kernel(
        np.array([1.0, 1.0]), 1.0, "rows"), [2.0, 2.0], rtol=1e-6)


@pytest.mark.parametrize("n,m,cl", [(512, 512, "6"), (512, 512, "8"), (130, 68, "0"), (37, 1024, "0"),
                                    (700, 300, "0")])
def test_batched_cluster_solver_matches_streaming_solver(otk, monkeypatch, n, m, cl):
    """K3c vs K3p on ragged shapes (rows not a multiple of the cluster, CTAs with no
    rows, several column chunks), warm start, fixed iterations and tolerance runs:
    same iteration counts and convergence, potentials within float32 rounding.
    K3c runs in the scaling domain (a stored stabilised kernel, FMA half-steps)
    and K3p in the log domain: each lands within ~3.5e-6 of the float64 oracle
    on these shapes (tools/k3_accuracy.py), so they agree to 5e-6."""
    rng = np.random.default_rng(n + m)
    B, d = 20, 5
    x = rng.standard_normal((B, n, d)).astype(np.float32)
    y = (rng.standard_normal((B, m, d)) + rng.uniform(-1, 1, (B, 1, d))).astype(np.float32)
    eps = np.array([0.05 * np.mean(np.sum((x[k, :64, None] - y[k, None, :64]) ** 2, -1))
                    for k in range(B)])
    g0 = (rng.standard_normal((B, m)) * eps[:, None]).astype(np.float32)
    monkeypatch.setenv("OTK_DENSE_CL", cl)
    for kw in (dict(threshold=1e-3, max_iters=500), dict(threshold=1e-300, max_iters=37),
               dict(threshold=1e-3, max_iters=500, g_init=g0)):
        monkeypatch.setenv("OTK_DENSE_KERNEL", "cluster")
        a = otk.solve_sinkhorn_batched(x, y, eps, **kw)
        monkeypatch.setenv("OTK_DENSE_KERNEL", "cta")
        b = otk.solve_sinkhorn_batched(x, y, eps, **kw)
        assert np.array_equal(a.iterations, b.iterations)
        assert np.array_equal(a.converged, b.converged)
        for k in range(B):
            assert rel_inf(a.f[k], b.f[k]) <= 5e-6
            assert rel_inf(a.g[k], b.g[k]) <= 5e-6


def _small_vs_general(otk, x, y, a, b, eps, **kw):
    """Run the one-kernel small solve and the launch-per-half-step loop on the
    same problem; return (outcome, outcome) where an outcome is the result or
    the (exception type, iteration / message) it raised."""
    from paper_2201_12324_b200 import _native as N

    def run(flags):
        g = otk.PointCloudGeometry(x, y)
        g.impl_flags = flags
        try:
            return otk.solve_sinkhorn(otk.LinearProblem(g, a, b), eps, **kw)
        except otk.DivergedError as e:
            return ("diverged", e.iteration)
        except ValueError as e:
            return ("value", str(e))
    return run(0), run(N.OTK_IMPL_NOPERSIST)


def test_persistent_small_solve_failure_paths_match_general_loop(otk):
    """The persistent small solve (per-CTA first-bad markers, one grid barrier
    per check) raises exactly what the general loop raises, at the same
    iteration: a warm start with NaN / +inf entries (reference geometry.py:65-72
    via apply_lse_kernel), and divergence from a zero-weight column whose
    kernel underflows (reference tests/test_sinkhorn.py:244-250 analog)."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((300, 3)).astype(np.float32)
    y = (rng.standard_normal((260, 3)) + 0.5).astype(np.float32)
    for bad in (np.nan, np.inf):
        g0 = np.zeros(260)
        g0[17] = bad
        fast, gen = _small_vs_general(otk, x, y, None, None, 0.5, g_init=g0)
        assert fast == gen and fast[0] == "value", (fast, gen)
    b = np.full(260, 1.0 / 259)
    b[-1] = 0.0
    y2 = y.copy()
    y2[-1] = 1e4  # far away: its column's kernel underflows at small eps
    fast, gen = _small_vs_general(otk, x, y2, None, b, 1e-3, inner_iters=1, max_iters=50)
    if isinstance(gen, tuple):
        assert fast == gen, (fast, gen)
    else:
        assert not isinstance(fast, tuple)
        assert fast.iterations == gen.iterations and fast.converged == gen.converged


@pytest.mark.parametrize("n,m", [(2048, 2048), (3000, 2100), (1, 7), (149, 150)])
def test_persistent_small_solve_shapes_and_zero_weights(otk, n, m):
    """Row-chunk shapes of the persistent small solve (one chunk per SM at the
    cfg1 size, several chunks per SM, a single row, chunk size 1-2) with zero
    weights on both sides (-inf potentials, empty rows / columns) against the
    general loop and the float64 oracle."""
    rng = np.random.default_rng(n + m)
    x = rng.standard_normal((n, 3)).astype(np.float32)
    y = (rng.standard_normal((m, 3)) * 1.3 + 0.2).astype(np.float32)
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.5, 1.5, m)
    if n > 1:
        a[::7] = 0.0
    b[::5] = 0.0
    a /= a.sum()
    b /= b.sum()
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = 0.05 * float(np.mean(geom64.cost_matrix()))
    ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-3, max_iters=300)
    fast, gen = _small_vs_general(otk, x, y, a, b, eps, threshold=1e-3, max_iters=300)
    for out in (fast, gen):
        assert out.iterations == ref["iterations"] and out.converged == ref["converged"]
        assert rel_inf(out.f, ref["f"]) <= POT_TOL
        assert rel_inf(out.g, ref["g"]) <= POT_TOL


@pytest.mark.parametrize("domain", ["scaled", "log"])
def test_batched_cluster_solver_edge_cases_match_oracle(otk, monkeypatch, domain):
    """K3c in both domains on the cases the scaling domain must fall back on:
    zero weights (dead columns and rows, -inf potentials), a far outlier
    column (its FMA partial underflows -> exact log-domain partial), a far-off
    warm start (kernel rebuilds) and a tight eps -- against the float64 oracle."""
    if domain == "log":
        monkeypatch.setenv("OTK_DENSE_DOMAIN", "log")
    rng = np.random.default_rng(77)
    B, n, m, d = 4, 300, 260, 4
    x = rng.standard_normal((B, n, d)).astype(np.float32)
    y = (rng.standard_normal((B, m, d)) + 0.3).astype(np.float32)
    y[1, 5] = 4.0  # far from every x (C/eps ~ 160): its scaled-domain partial underflows
    a = rng.uniform(0.5, 1.5, (B, n))
    b = rng.uniform(0.5, 1.5, (B, m))
    a[2, ::11] = 0.0
    b[2, ::7] = 0.0
    a /= a.sum(axis=1, keepdims=True)
    b /= b.sum(axis=1, keepdims=True)
    Cs = [((x[k].astype(np.float64)[:, None] - y[k].astype(np.float64)[None]) ** 2).sum(-1) for k in range(B)]
    eps = np.array([0.05 * C.mean() for C in Cs])
    eps[3] *= 0.2
    g0 = np.zeros((B, m), np.float32)
    g0[0] = (rng.standard_normal(m) * 60 * eps[0]).astype(np.float32)  # drifts far: rebuilds
    outs = otk.solve_sinkhorn_batched(x, y, eps, a, b, threshold=1e-300, max_iters=40, g_init=g0)
    for k in range(B):
        ref = oracle.sinkhorn(oracle.DenseOracle(Cs[k].astype(np.float32).astype(np.float64)), a[k], b[k],
                              float(eps[k]), threshold=1e-300, max_iters=40, g_init=g0[k].astype(np.float64))
        assert outs.iterations[k] == ref["iterations"]
        assert rel_inf(outs.f[k], ref["f"]) <= POT_TOL, (k, rel_inf(outs.f[k], ref["f"]))
        assert rel_inf(outs.g[k], ref["g"]) <= POT_TOL, (k, rel_inf(outs.g[k], ref["g"]))


@pytest.mark.parametrize("d,cost_fn", [(3, "sqeucl"), (6, "sqeucl"), (12, "sqeucl"), (3, "eucl"),
                                       (21, "eucl"), (48, "sqeucl"), (67, "sqeucl")])
def test_persistent_small_solve_stored_kernel_edge_cases(otk, monkeypatch, d, cost_fn):
    """The stored-kernel half-steps of the persistent small solve (exps taken
    once, FP32 matrix-vector half-steps, csrc/solve_small.cu) on the cases that
    send a CTA back to its exact passes or sit at the edge of the scaling
    window: a far-off warm start (columns drift > 40 bits -> rebuilds), a tight
    eps, zero weights on both sides (-inf potentials), one far outlier point --
    against the float64 oracle and against the same kernel with the stored
    path switched off (OTK_SMALL_STORED=0)."""
    rng = np.random.default_rng(300 + d)
    n, m = 1500, 1333
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.3).astype(np.float32)
    y[5] = 4.0
    a = rng.uniform(0.5, 1.5, n)
    b = rng.uniform(0.5, 1.5, m)
    a[::11] = 0.0
    b[::7] = 0.0
    a /= a.sum()
    b /= b.sum()
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64), cost_fn=cost_fn)
    eps = 0.02 * float(np.mean(geom64.cost_matrix()))
    g0 = (rng.standard_normal(m) * 60 * eps).astype(np.float32)
    ref = oracle.sinkhorn(geom64, a, b, eps, threshold=1e-300, max_iters=40, g_init=g0.astype(np.float64))

    def run():
        prob = otk.LinearProblem(otk.PointCloudGeometry(x, y, cost_fn=cost_fn), a, b)
        return otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=40, g_init=g0)
    stored, stored2 = run(), run()
    if d > 19:  # no plain small solve beyond 19 coordinates: compare with the general loop instead
        from paper_2201_12324_b200 import _native as N

        def run():  # noqa: F811
            geom = otk.PointCloudGeometry(x, y, cost_fn=cost_fn)
            geom.impl_flags = N.OTK_IMPL_NOPERSIST
            return otk.solve_sinkhorn(otk.LinearProblem(geom, a, b), eps, threshold=1e-300, max_iters=40,
                                      g_init=g0)
    else:
        monkeypatch.setenv("OTK_SMALL_STORED", "0")
    plain = run()
    for out in (stored, plain):
        assert out.iterations == ref["iterations"] and len(out.errors) == len(ref["errors"])
        assert rel_inf(out.f, ref["f"]) <= POT_TOL, rel_inf(out.f, ref["f"])
        assert rel_inf(out.g, ref["g"]) <= POT_TOL, rel_inf(out.g, ref["g"])
        np.testing.assert_allclose(out.dual_trace, ref["dual_trace"], rtol=1e-5)
    assert np.array_equal(stored.f, stored2.f) and np.array_equal(stored.g, stored2.g)
    assert rel_inf(stored.f, plain.f) <= 1e-5 and rel_inf(stored.g, plain.g) <= 1e-5


def test_persistent_small_solve_stored_kernel_long_run_has_no_gauge_drift(otk, monkeypatch):
    """Sinkhorn does not contract the (f + c, g - c) direction, so a bias that
    repeats identically every half-step adds up linearly with the iterations.
    The stored-kernel half-steps evaluate ex2 / lg2 at frozen arguments; the
    tighter drift window at later checks (DRIFT_CHECK, csrc/solve_small.cu)
    rebuilds the terms once the potentials have settled.  600 forced
    iterations of a small, large-eps problem (few columns to average over,
    potentials of a few bits): stored and plain kernels against the oracle."""
    rng = np.random.default_rng(5)
    n, m, d = 48, 40, 3
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.5).astype(np.float32)
    geom64 = oracle.PointCloudOracle(x.astype(np.float64), y.astype(np.float64))
    eps = 0.5 * float(np.mean(geom64.cost_matrix()))
    ref = oracle.sinkhorn(geom64, None, None, eps, threshold=1e-300, max_iters=600)
    prob = otk.LinearProblem(otk.PointCloudGeometry(x, y))
    stored = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=600)
    monkeypatch.setenv("OTK_SMALL_STORED", "0")
    plain = otk.solve_sinkhorn(prob, eps, threshold=1e-300, max_iters=600)
    for out in (stored, plain):
        # an exact float32 fixed point (marginal error 0.0) may end the loop early: same potentials
        assert out.iterations == 600 or (out.converged and out.errors[-1] == 0.0)
        assert rel_inf(out.f, ref["f"]) <= 2e-5, rel_inf(out.f, ref["f"])
        assert rel_inf(out.g, ref["g"]) <= 2e-5, rel_inf(out.g, ref["g"])


@pytest.mark.parametrize("route", ["small", "general", "batched"])
def test_fixed_iters_runs_every_iteration_past_an_exact_fixed_point(otk, route):
    """float32 iterates can reach an exact fixed point (f_{t+1} == f_t bitwise, marginal
    error 0.0), which satisfies any positive threshold and ends the loop as the
    reference's test `err <= threshold` (sinkhorn.py:187) says.  The measurement knob
    `fixed_iters` keeps iterating: same potentials, every check recorded, converged False."""
    from paper_2201_12324_b200 import _native as N
    wl = workloads.cfg1(n=300, m=260)
    iters = 400
    if route == "batched":
        x, y = wl.x[None], wl.y[None]
        stop = otk.solve_sinkhorn_batched(x, y, wl.eps, threshold=1e-300, max_iters=iters)[0]
        full = otk.solve_sinkhorn_batched(x, y, wl.eps, threshold=1e-300, max_iters=iters, fixed_iters=True)[0]
    else:
        geom = otk.PointCloudGeometry(wl.x, wl.y)
        if route == "general":
            geom.impl_flags = N.OTK_IMPL_NOPERSIST
        prob = otk.LinearProblem(geom)
        stop = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=iters)
        full = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=iters, fixed_iters=True)
    assert full.iterations == iters and not full.converged and len(full.errors) == iters // 10
    if stop.converged:  # an exact fixed point: nothing moves afterwards
        assert stop.errors[-1] == 0.0 and stop.iterations < iters
        assert np.array_equal(stop.f, full.f) and np.array_equal(stop.g, full.g)
        assert full.errors[-1] == 0.0
    else:
        assert stop.iterations == iters
