"""The ``lin`` CLI (reference otkit/cli.py:123-172).

CPU: argument / input validation and exit codes (no device touched).
GPU: the CLI's JSON equals the library calls it wraps (reference acceptance
criterion 12, test_acceptance.py:377-466) and the oracle within tolerance;
the coupling CSV round-trips; exit code 2 when not converged.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2201_12324_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write(path, arr):
    np.savetxt(path, np.atleast_2d(arr), delimiter=",")
    return str(path)


def test_input_errors_exit_1(tmp_path, capsys):
    assert cli.main(["lin", "--x", "nope.csv"]) == 1                 # needs x and y
    x = _write(tmp_path / "x.csv", np.zeros((3, 2)))
    y = _write(tmp_path / "y.csv", np.zeros((4, 2)))
    assert cli.main(["lin", "--x", x, "--y", y, "--eps", "1", "--eps-rel", "1"]) == 1
    assert cli.main(["lin", "--x", x, "--y", y, "--solver", "lr"]) == 1
    bad = _write(tmp_path / "a.csv", np.array([0.5, 0.6, 0.1]))
    assert cli.main(["lin", "--x", x, "--y", y, "--a", bad]) == 1    # sums to 1.2
    assert cli.main(["lin", "--x", str(tmp_path / "missing.csv"), "--y", y]) == 1
    assert cli.main(["quad", "--x", x, "--y", y]) == 1
    assert cli.main(["lin", "--bogus"]) == 1
    assert "error:" in capsys.readouterr().err


def test_weights_rescaled_within_1e6():
    w = cli._as_cli_weights(np.array([0.25, 0.25, 0.5 + 5e-7]), 3, "a")
    assert w.sum() == pytest.approx(1.0, abs=1e-15)


@pytest.mark.gpu
def test_cli_matches_library_and_oracle(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as otk
    rng = np.random.default_rng(12)
    x = rng.standard_normal((60, 3))
    y = rng.standard_normal((45, 3)) + 0.5
    a = rng.uniform(0.5, 1.5, 60)
    a /= a.sum()
    xp, yp, ap = _write(tmp_path / "x.csv", x), _write(tmp_path / "y.csv", y), _write(tmp_path / "a.csv", a)
    out_json, plan_csv = tmp_path / "out.json", tmp_path / "plan.csv"
    rc = subprocess.run([sys.executable, "-m", "paper_2201_12324_b200", "lin", "--x", xp, "--y", yp,
                         "--a", ap, "--eps-rel", "0.05", "--out", str(out_json),
                         "--coupling-out", str(plan_csv)], cwd=ROOT).returncode
    assert rc == 0
    got = json.loads(out_json.read_text())
    # the library calls the CLI wraps, on the same parsed inputs
    xr, yr = cli.read_matrix(xp), cli.read_matrix(yp)
    geom = otk.PointCloudGeometry(xr, yr)
    prob = otk.LinearProblem(geom, cli._as_cli_weights(cli.read_vector(ap), 60, "a"))
    eps = 0.05 * geom.mean_cost()
    out = otk.solve_sinkhorn(prob, eps)
    cost = otk.reg_ot_cost(out, prob)
    assert got == {"command": "lin", "solver": "sinkhorn", "transport_cost": cost.transport_cost,
                   "dual_objective": cost.dual_objective, "iterations": out.iterations,
                   "converged": out.converged, "eps": out.eps}
    plan = cli.read_matrix(str(plan_csv))
    np.testing.assert_allclose(plan, otk.transport_matrix(out, prob).matrix, rtol=0, atol=0)
    # and the oracle (reference restatement) on the same inputs
    ref = oracle.sinkhorn(oracle.PointCloudOracle(xr, yr), prob.a, None, eps)
    tc, dual = oracle.reg_ot_cost(oracle.PointCloudOracle(xr, yr), ref["f"], ref["g"], prob.a,
                                  np.full(45, 1 / 45), eps)
    assert got["iterations"] == ref["iterations"]
    assert abs(got["transport_cost"] - tc) <= 1e-5 * abs(tc)
    # not converged -> exit code 2
    rc = subprocess.run([sys.executable, "-m", "paper_2201_12324_b200", "lin", "--x", xp, "--y", yp,
                         "--eps-rel", "0.05", "--max-iters", "3", "--out", str(out_json)],
                        cwd=ROOT).returncode
    assert rc == 2 and json.loads(out_json.read_text())["converged"] is False


def test_barycenter_input_errors_exit_1(tmp_path, capsys):
    s = _write(tmp_path / "s.csv", np.linspace(0, 1, 5)[:, None])
    h = _write(tmp_path / "h.csv", np.full(5, 0.2))
    bad = _write(tmp_path / "bad.csv", np.full(5, 0.3))
    short = _write(tmp_path / "short.csv", np.full(4, 0.25))
    assert cli.main(["barycenter", "--hist", h]) == 1                       # no support / grid
    assert cli.main(["barycenter", "--grid", s, "--hist", h]) == 1          # grid not in build
    assert cli.main(["barycenter", "--support", s, "--hist", bad]) == 1     # sums to 1.5
    assert cli.main(["barycenter", "--support", s, "--hist", short]) == 1   # wrong length
    assert cli.main(["barycenter", "--support", s, "--hist", h, "--hist", h,
                     "--weights", "0.5,x"]) == 1
    assert cli.main(["barycenter", "--support", s, "--hist", h, "--hist", h,
                     "--weights", "0.5,0.6"]) == 1
    assert cli.main(["barycenter", "--support", s, "--hist", h, "--eps", "1",
                     "--eps-rel", "1"]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_barycenter_cli_matches_library(tmp_path, capsys):
    """Reference test_cli.py:231-266 intent: the CLI JSON and CSV equal the library call."""
    import paper_2201_12324_b200 as otk
    pts = np.linspace(0.0, 1.0, 11)
    h1, h2 = np.zeros(11), np.zeros(11)
    h1[2] = 1.0
    h2[8] = 1.0
    support = _write(tmp_path / "support.csv", pts[:, None])
    out_path = tmp_path / "bary.csv"
    code = cli.main(["barycenter", "--support", support, "--hist", _write(tmp_path / "h1.csv", h1),
                     "--hist", _write(tmp_path / "h2.csv", h2), "--weights", "0.5,0.5",
                     "--eps-rel", "1e-3", "--barycenter-out", str(out_path)])
    payload = json.loads(capsys.readouterr().out)
    assert code == 0
    geom = otk.PointCloudGeometry(pts[:, None], pts[:, None])
    out = otk.solve_barycenter(otk.BarycenterProblem(geom, np.stack([h1, h2]), np.array([0.5, 0.5])),
                               1e-3 * geom.mean_cost())
    assert payload["barycenter"] == out.barycenter.tolist()
    assert payload["iterations"] == out.iterations
    np.testing.assert_array_equal(np.loadtxt(out_path, delimiter=","), out.barycenter)
    assert int(np.argmax(out.barycenter)) == 5
