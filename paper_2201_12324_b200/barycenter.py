"""Fixed-support Wasserstein barycenters on the GPU.

Drop-in for reference otkit/barycenter.py: same names (``BarycenterProblem``,
``BarycenterOutput``, ``solve_barycenter``), same validation
(barycenter.py:39-64, 96-106), same iteration, stopping rule and
``DivergedError`` (barycenter.py:107-133).  The K histograms share one
square support geometry; the solve is ONE cooperative kernel launch
(csrc/bary.cu, ``otk_solve_barycenter``) over the support cost materialised
once on the device (C and C^T, 8 N^2 bytes, padded rows).  ``PointCloudGeometry``
(sqeucl / eucl / cosine) and ``DenseGeometry`` supports are accepted;
``GridGeometry`` (separable grids) is not part of this build.
"""

from __future__ import annotations

import dataclasses
import logging

import numpy as np

from . import _native as N
from ._device import as_device_f32, device, stream
from .errors import DivergedError
from .geometry import DenseGeometry, Geometry, PointCloudGeometry

logger = logging.getLogger(__name__)

__all__ = ["BarycenterProblem", "BarycenterOutput", "solve_barycenter"]

_LOG2E = 1.4426950408889634


@dataclasses.dataclass(frozen=True, eq=False)
class BarycenterProblem:
    """K histograms on one support plus barycentric weights (barycenter.py:26-64).

    ``geom`` must be square (support against itself); ``histograms`` is a
    (K, N) array of probability vectors; ``weights`` (K,) defaults to uniform.
    """

    geom: Geometry
    histograms: np.ndarray
    weights: np.ndarray | None = None

    def __post_init__(self):
        n, m = self.geom.shape
        if n != m:
            raise ValueError(f"barycenter geometry must be square, got shape {(n, m)}")
        hists = np.atleast_2d(np.asarray(self.histograms, dtype=float))
        if hists.shape[1] != n:
            raise ValueError(f"histograms must have {n} columns, got {hists.shape[1]}")
        if hists.shape[0] < 1:
            raise ValueError("need at least one histogram")
        if not np.all(np.isfinite(hists)) or np.any(hists < 0):
            raise ValueError("histograms must be entrywise finite and nonnegative")
        if np.any(np.abs(hists.sum(axis=1) - 1.0) > 1e-8):
            raise ValueError("each histogram must sum to 1")
        k = hists.shape[0]
        if self.weights is None:
            weights = np.full(k, 1.0 / k)
        else:
            weights = np.asarray(self.weights, dtype=float)
            if weights.shape != (k,):
                raise ValueError(f"weights must have shape ({k},), got {weights.shape}")
            if not np.all(np.isfinite(weights)) or np.any(weights < 0):
                raise ValueError("weights must be entrywise finite and nonnegative")
            if abs(weights.sum() - 1.0) > 1e-8:
                raise ValueError("weights must sum to 1")
        object.__setattr__(self, "histograms", hists)
        object.__setattr__(self, "weights", weights)


@dataclasses.dataclass(frozen=True)
class BarycenterOutput:
    """barycenter.py:67-72, plus the per-iteration marginal errors (extension)."""

    barycenter: np.ndarray
    converged: bool
    iterations: int
    eps: float
    errors: np.ndarray | None = dataclasses.field(default=None, repr=False, compare=False)


def _support_costs(geom):
    """(C_p, C^T_p) of the square support on the device: fp32 row-major with the
    leading dimension padded to a multiple of 4 by +inf costs (otk_barycenter_pad)."""
    import torch
    lib = N.lib()
    n = geom.shape[0]
    if isinstance(geom, DenseGeometry):
        C = geom._c()
    elif isinstance(geom, PointCloudGeometry):
        px, py = geom._points()  # centred kernel points (geometry.centered_points)
        C = torch.empty((n, n), dtype=torch.float32, device=px.device)
        N.check(lib.otk_dense_cost(N.ptr(px), N.ptr(py), 1, n, n, px.shape[1],
                                   geom._cost_flags, N.ptr(C),
                                   None, stream()), "barycenter support cost")
    else:
        raise TypeError(f"solve_barycenter supports PointCloudGeometry and DenseGeometry, "
                        f"got {type(geom).__name__}")
    ld = int(lib.otk_barycenter_ld(n))
    Cp = torch.empty((n, ld), dtype=torch.float32, device=C.device)
    CTp = torch.empty_like(Cp)
    N.check(lib.otk_barycenter_pad(N.ptr(C), n, ld, N.ptr(Cp), N.ptr(CTp), stream()),
            "barycenter_pad")
    return Cp, CTp, ld


def _check_memory(n: int, k: int) -> None:
    import torch
    need = 12 * n * (n + 4) + 12 * k * (n + 4) + 64 * n
    free, _ = torch.cuda.mem_get_info()
    if need > 0.9 * free:
        raise ValueError(f"barycenter support of {n} points needs {need / 2**30:.1f} GiB of "
                         f"device memory for its cost (C and C^T); {free / 2**30:.1f} GiB free")


def solve_barycenter(bp: BarycenterProblem, eps: float | None = None, *,
                     threshold: float = 1e-4, max_iters: int = 1000) -> BarycenterOutput:
    """Scaling iterations until every coupling's barycenter-side marginal is within
    ``threshold`` (L1, max over histograms) of the current p (barycenter.py:75-133).

    Raises:
      DivergedError: on NaN in log p (eps too small to couple the support).
    """
    import torch
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    if not (threshold > 0):
        raise ValueError("threshold must be positive")
    geom = bp.geom
    if eps is None:
        eps = geom.epsilon_default
    eps = float(eps)
    if not (eps > 0):
        raise ValueError("eps must be positive")
    with np.errstate(over="ignore"):
        kappa = np.float32(_LOG2E / eps)
    if not np.isfinite(kappa):
        raise ValueError(f"eps={eps!r} is below the range of the fp32 device kernels")
    k, n = bp.histograms.shape
    dev = device()
    _check_memory(n, k)
    C, CT, ld = _support_costs(geom)
    with np.errstate(divide="ignore"):
        log2h = torch.as_tensor(np.ascontiguousarray(np.log2(bp.histograms), dtype=np.float32),
                                device=dev)
    w = torch.as_tensor(bp.weights, dtype=torch.float64, device=dev)
    lib = N.lib()
    plen = int(lib.otk_barycenter_part_len(n, k))
    if plen <= 0:
        raise RuntimeError("otk_barycenter_part_len failed")
    F = torch.empty((k, ld), dtype=torch.float32, device=dev)
    G = torch.empty_like(F)
    B = torch.empty_like(F)
    lp2 = torch.empty(n, dtype=torch.float64, device=dev)
    errors = torch.full((max_iters,), float("nan"), dtype=torch.float64, device=dev)
    state = torch.zeros(8, dtype=torch.int32, device=dev)
    part = torch.empty(plen, dtype=torch.float64, device=dev)
    N.check(lib.otk_solve_barycenter(N.ptr(C), N.ptr(CT), n, ld, k, N.ptr(log2h), N.ptr(w), eps,
                                     float(threshold), int(max_iters), N.ptr(F), N.ptr(G),
                                     N.ptr(B), N.ptr(lp2), N.ptr(errors), N.ptr(state),
                                     N.ptr(part), stream()), "solve_barycenter")
    iters, converged, nan_iter, _grid = (int(v) for v in state.cpu().numpy()[:4])
    if nan_iter:
        raise DivergedError("NaN in barycenter iterations; eps is likely too small",
                            iteration=nan_iter)
    if not converged:
        logger.info("barycenter: no convergence after %d iterations", iters)
    log2p = lp2.cpu().numpy()
    p = np.exp2(log2p - np.max(log2p))
    return BarycenterOutput(barycenter=p / p.sum(), converged=bool(converged), iterations=iters,
                            eps=eps, errors=errors.cpu().numpy()[:iters])
