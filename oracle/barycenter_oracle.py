"""CPU oracle for fixed-support barycenters (TEST INFRASTRUCTURE ONLY).

float64 numpy restatement of the reference's iterative Bregman projections,
otkit/barycenter.py:73-133 (solve_barycenter) with the problem checks of
barycenter.py:39-64 (BarycenterProblem.__post_init__).  Used by tests/ as
the checker for the CUDA path (csrc/bary.cu); pinned against fixtures the
reference itself wrote (tests/golden/make_golden.py -> barycenter.npz).
The product package never imports it.
"""

from __future__ import annotations

import numpy as np

from .sinkhorn_oracle import OracleDiverged, OracleValueError


def check_problem(geom, histograms, weights=None):
    """barycenter.py:39-64: square geometry, (K, N) probability rows, weights on the simplex."""
    n, m = geom.shape
    if n != m:
        raise OracleValueError(f"barycenter geometry must be square, got shape {(n, m)}")
    hists = np.atleast_2d(np.asarray(histograms, dtype=float))
    if hists.shape[1] != n:
        raise OracleValueError(f"histograms must have {n} columns")
    if not np.all(np.isfinite(hists)) or np.any(hists < 0):
        raise OracleValueError("histograms must be entrywise finite and nonnegative")
    if np.any(np.abs(hists.sum(axis=1) - 1.0) > 1e-8):
        raise OracleValueError("each histogram must sum to 1")
    k = hists.shape[0]
    if weights is None:
        w = np.full(k, 1.0 / k)
    else:
        w = np.asarray(weights, dtype=float)
        if w.shape != (k,) or not np.all(np.isfinite(w)) or np.any(w < 0):
            raise OracleValueError("bad barycentric weights")
        if abs(w.sum() - 1.0) > 1e-8:
            raise OracleValueError("weights must sum to 1")
    return hists, w


def solve_barycenter(geom, histograms, weights, eps, threshold=1e-4, max_iters=1000):
    """barycenter.py:96-133.  Returns (p normalised, converged, iterations, log_p).

    Per iteration t and histogram k (log domain, zeros allowed):
        f_k    = eps log h_k - LSE_rows(0, g_k)          (barycenter.py:117)
        back_k = LSE_cols(f_k, 0)                        (barycenter.py:118)
        log p  = sum_k w_k back_k / eps                  (barycenter.py:119)
        NaN in log p -> diverged at t                    (barycenter.py:120-121)
        err    = max_k |exp(LSE_cols(f_k, g_k)/eps) - p|_1   (barycenter.py:123-126)
        g_k    = eps log p - back_k                      (barycenter.py:127-128)
    stopping once err <= threshold (barycenter.py:129-131).
    """
    hists, w = check_problem(geom, histograms, weights)
    if max_iters < 1:
        raise OracleValueError("max_iters must be >= 1")
    if not threshold > 0:
        raise OracleValueError("threshold must be positive")
    eps = float(eps)
    if not eps > 0:
        raise OracleValueError("eps must be positive")
    k, n = hists.shape
    with np.errstate(divide="ignore"):
        log_h = np.log(hists)
    zeros = np.zeros(n)
    f = np.zeros((k, n))
    g = np.zeros((k, n))
    back = np.zeros((k, n))
    log_p = np.full(n, -np.log(n))
    converged = False
    t = 0
    for t in range(1, max_iters + 1):
        for i in range(k):
            f[i] = eps * log_h[i] - geom.apply_lse_kernel(zeros, g[i], eps, "rows")
            back[i] = geom.apply_lse_kernel(f[i], zeros, eps, "cols")
        log_p = (w @ back) / eps
        if np.isnan(log_p).any():
            raise OracleDiverged(t)
        p = np.exp(log_p)
        err = 0.0
        for i in range(k):
            marginal = np.exp(geom.apply_lse_kernel(f[i], g[i], eps, "cols") / eps)
            err = max(err, float(np.abs(marginal - p).sum()))
        for i in range(k):
            g[i] = eps * log_p - back[i]
        if err <= threshold:
            converged = True
            break
    p = np.exp(log_p)
    return p / p.sum(), converged, t, log_p
