"""CPU-only checks: the C ABI library loads and exports what include/otk.h
declares, and the host-side validation mirrors the reference (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "otk.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(otk_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def native():
    from paper_2201_12324_b200 import _build, _native
    if not os.path.exists(_native.lib_path()):
        _build.build()
    return _native


def test_library_exports_every_header_symbol(native):
    lib = native.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/otk.h but not exported"
        assert s in native.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.otk_abi_version() == native.ABI_VERSION


def test_library_is_sm100a(native):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", native.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_solve_args_layout_matches_header(native):
    import ctypes
    A = native.SolveArgs
    # spot-check natural alignment of the struct mirror
    assert A.eps_target.offset % 8 == 0 and A.workspace.offset % 8 == 0
    assert ctypes.sizeof(A) % 8 == 0


def test_geometry_validation_matches_reference():
    import paper_2201_12324_b200 as otk
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.zeros((2, 2)), np.zeros((2, 3)))
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.zeros((2, 1)), np.zeros((2, 1)), "manhattan")
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.zeros((0, 1)), np.zeros((2, 1)))
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.array([[np.inf]]), np.zeros((2, 1)))
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.zeros((2, 1)), np.zeros((2, 1)), block_size=0)
    with pytest.raises(ValueError):
        otk.DenseGeometry(np.array([[np.inf]]))
    g = otk.PointCloudGeometry(np.zeros((3, 1)), np.zeros((3, 1)))
    with pytest.raises(ValueError, match="entries"):
        g.cost_matrix(max_entries=8)
    with pytest.raises(ValueError):
        g.apply_lse_kernel(np.zeros(3), np.zeros(3), 1.0, "diagonal")
    x = np.zeros((4, 2))
    assert otk.PointCloudGeometry(x, x)._same_points
    assert otk.PointCloudGeometry(x, x.copy())._same_points


@pytest.mark.parametrize("kwargs", [
    {"target": 0.0}, {"target": 1.0, "init_scale": 0.5}, {"target": 1.0, "decay": 0.0},
    {"target": 1.0, "decay": 1.5}, {"target": 1.0, "init_scale": 10.0, "decay": 1.0}])
def test_epsilon_schedule_rejects_bad_parameters(kwargs):
    import paper_2201_12324_b200 as otk
    with pytest.raises(ValueError):
        otk.EpsilonSchedule(**kwargs)


def test_epsilon_schedule_values():
    import paper_2201_12324_b200 as otk
    s = otk.EpsilonSchedule(0.01, init_scale=100.0, decay=0.5)
    assert s.at(0) == 1.0 and s.at(1) == 0.5 and s.at(50) == 0.01


@pytest.mark.parametrize("a,b", [(np.array([0.5, 0.6]), None), (np.array([-0.1, 1.1]), None),
                                 (None, np.array([1.0]))])
def test_linear_problem_rejects_invalid_weights(a, b):
    import paper_2201_12324_b200 as otk
    with pytest.raises(ValueError):
        otk.LinearProblem(otk.DenseGeometry(np.zeros((2, 2))), a, b)


def test_solver_rejects_bad_arguments_before_touching_the_gpu():
    import paper_2201_12324_b200 as otk
    prob = otk.LinearProblem(otk.DenseGeometry(np.ones((2, 2))))
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 0.0)
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 1.0, threshold=0.0)
    with pytest.raises(ValueError):
        otk.solve_sinkhorn(prob, 1.0, max_iters=0)
    with pytest.raises(otk.DivergedError) as exc:
        otk.solve_sinkhorn(prob, 1e-320, inner_iters=1)
    assert exc.value.iteration == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2201_12324_b200 as otk
    prob = otk.LinearProblem(otk.PointCloudGeometry(np.zeros((3, 2)), np.ones((3, 2))))
    with pytest.raises(RuntimeError, match="CUDA"):
        otk.solve_sinkhorn(prob, 1.0)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2201_12324_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith(".py"):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), fn


def test_cosine_and_apply_kernel_validation_like_reference():
    """test_geometry.py:211-223: zero vectors with cosine, bad axis / lengths /
    eps for apply_kernel -- all raised before any device work."""
    import paper_2201_12324_b200 as otk
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.array([[0.0, 0.0]]), np.array([[1.0, 0.0]]), "cosine")
    with pytest.raises(ValueError):
        otk.PointCloudGeometry(np.ones((2, 2)), np.ones((2, 2)), "manhattan")
    assert otk.PointCloudGeometry(np.ones((2, 2)), np.ones((2, 2)), "eucl").cost_fn == "eucl"
    geom = otk.DenseGeometry(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        geom.apply_kernel(np.ones(3), 1.0, "diagonal")
    with pytest.raises(ValueError):
        geom.apply_kernel(np.ones(2), 1.0, "rows")
    with pytest.raises(ValueError):
        geom.apply_kernel(np.ones(3), 0.0, "rows")
