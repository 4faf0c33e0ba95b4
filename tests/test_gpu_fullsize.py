"""Whole solves at the FULL BASELINE sizes vs the unmodified reference (needs a B200).

The fixtures come from tests/golden/make_fullsize_golden.py, which runs the
reference's own `solve_sinkhorn` loop (sinkhorn.py:151-200) over its own
`PointCloudGeometry.apply_lse_kernel` (geometry.py:336-354) evaluated on
256-aligned row/column chunks in worker processes, and `reg_ot_cost`
(sinkhorn.py:210-216) in 256-row blocks.  Inputs regenerate from
workloads.py (deterministic numpy draws).  Every solve here runs on the
default routing -- tcgen05 half-steps, anchored from the second half-step of
each role (they are >= 2^27 cells), CTA-pair MMA at d = 128, V4 accumulators
at d = 1024 -- i.e. the kernels bench.py times.

Tolerances (north_star): f, g 1e-4 relative (inf-norm); transport cost and
dual 1e-5 relative; identical iteration count and converged flag.  The
marginal errors and the dual trace are the reference's check values
(sinkhorn.py:183-186) evaluated by the fused check kernel from float32
potentials with float64 sums: errors within 1e-3 relative plus four times the
float32 floor ulp(max|f|)/eps (each row's r_i = a_i exp((f_i - f'_i)/eps)
carries a relative rounding of that size; ~6e-6 for cfg5),
dual trace within 1e-5 relative.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_2201_12324_b200 import workloads

pytestmark = pytest.mark.gpu

POT_TOL = 1e-4
COST_TOL = 1e-5
ERR_RTOL = 1e-3


def err_floor(f, eps):
    """float32 floor of the marginal error: ulp(max|f|) / eps."""
    return float(np.spacing(np.float32(np.max(np.abs(f))))) / float(eps)


@pytest.fixture(scope="module")
def otk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as m
    from paper_2201_12324_b200 import _native
    _native.lib()
    return m


_WL = {}


def workload(k):
    if k not in _WL:
        _WL.clear()
        _WL[k] = workloads.make(k)
    return _WL[k]


def rel_inf(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / np.max(np.abs(want)))


def _check_against(otk, fx, out, prob):
    assert out.iterations == int(fx["iterations"])
    assert out.converged == bool(fx["converged"])
    assert len(out.errors) == len(fx["errors"]) and len(out.dual_trace) == len(fx["dual_trace"])
    ef, eg = rel_inf(out.f, fx["f"]), rel_inf(out.g, fx["g"])
    assert ef <= POT_TOL and eg <= POT_TOL, (ef, eg)
    np.testing.assert_allclose(out.errors, fx["errors"], rtol=ERR_RTOL,
                               atol=4.0 * err_floor(fx["f"], fx["eps"]))
    np.testing.assert_allclose(out.dual_trace, fx["dual_trace"], rtol=COST_TOL)
    cost = otk.reg_ot_cost(out, prob)
    rt = abs(cost.transport_cost / float(fx["transport"]) - 1.0)
    rd = abs(cost.dual_objective / float(fx["dual"]) - 1.0)
    assert rt <= COST_TOL and rd <= COST_TOL, (rt, rd)
    return ef, eg, rt, rd


def _fixtures(prefix):
    names = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".npz"))
    return names


@pytest.mark.parametrize("name", _fixtures("full_cfg2") + _fixtures("full_cfg4") + _fixtures("full_cfg5"))
def test_full_size_solve_matches_reference(otk, name):
    """Fixed-iteration (threshold 1e-300, check at t == max_iters) and
    to-tolerance solves of cfg2 / cfg4 / cfg5 at their BASELINE sizes."""
    fx = load_golden(name)
    k = int(name.split("cfg")[1][0])
    wl = workload(k)
    assert float(fx["eps"]) == wl.eps
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    out = otk.solve_sinkhorn(prob, wl.eps, threshold=float(fx.get("threshold", 1e-300)),
                             max_iters=int(fx["max_iters"]))
    _check_against(otk, fx, out, prob)


def test_cfg3_all_512_problems_match_reference(otk):
    """The one-launch batched solve (K3c, default) on the whole cfg3 batch vs
    the reference's DenseGeometry solve of every problem."""
    fx = load_golden("full_cfg3_all")
    wl = workloads.cfg3()
    np.testing.assert_array_equal(wl.eps, fx["eps"])
    outs, costs = otk.solve_sinkhorn_batched(wl.x, wl.y, wl.eps, threshold=wl.threshold,
                                             max_iters=wl.max_iters, return_cost=True)
    np.testing.assert_array_equal(outs.iterations, fx["iterations"])
    np.testing.assert_array_equal(outs.converged, fx["converged"])
    df = np.max(np.abs(outs.f - fx["f"]), axis=1) / fx["f_absmax"]
    dg = np.max(np.abs(outs.g - fx["g"]), axis=1) / fx["g_absmax"]
    assert df.max() <= POT_TOL and dg.max() <= POT_TOL, (df.max(), dg.max())
    costs = np.asarray(costs, np.float64)
    np.testing.assert_allclose(costs[:, 0], fx["transport"], rtol=COST_TOL)
    np.testing.assert_allclose(costs[:, 1], fx["dual"], rtol=COST_TOL)
    for k in range(0, 512, 37):  # the per-problem check traces
        nk = int(fx["n_checks"][k])
        np.testing.assert_allclose(outs[k].errors, fx["errors"][k, :nk], rtol=ERR_RTOL,
                                   atol=4.0 * err_floor(fx["f"][k], fx["eps"][k]))
        np.testing.assert_allclose(outs[k].dual_trace, fx["dual_trace"][k, :nk], rtol=COST_TOL)


@pytest.mark.parametrize("name", _fixtures("conv_cfg"))
def test_converged_flag_pinned_by_float64_check(otk, name):
    """The GPU's converged flag at full size, pinned by the reference's check
    pass evaluated in float64 at the potentials a GPU run converged with
    (make_fullsize_golden.py conv mode): the same solve today reproduces those
    potentials, and the float64 marginal error at them is below the threshold."""
    fx = load_golden(name)
    k = int(name.split("cfg")[1][0])
    wl = workload(k)
    prob = otk.LinearProblem(otk.PointCloudGeometry(wl.x, wl.y), wl.a, wl.b)
    out = otk.solve_sinkhorn(prob, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
    assert out.converged and out.iterations == int(fx["iterations"])
    assert rel_inf(out.f, fx["f"]) <= 1e-5 and rel_inf(out.g, fx["g"]) <= 1e-5
    assert float(fx["ref_error"]) <= wl.threshold
    np.testing.assert_allclose(out.errors[-1], float(fx["ref_error"]), rtol=ERR_RTOL,
                               atol=4.0 * err_floor(fx["f"], fx["eps"]))
