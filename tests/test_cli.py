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
    assert cli.main(["lin", "--x", x, "--y", y, "--cost", "eucl"]) == 1
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
