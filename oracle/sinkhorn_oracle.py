"""Float64 numpy restatement of the reference Sinkhorn path (TEST INFRASTRUCTURE ONLY).

Restates, in this repo's own code, the arithmetic of the reference package
``otkit`` (paths relative to /root/reference/pkg/src/otkit):

* ``logsumexp``            -- the third-party ``scipy.special.logsumexp``
  (``scipy>=1.9`` pinned at pkg/pyproject.toml:12; 1.18.1 in this image)
  called at geometry.py:211,347,353.  Published algorithm: shift by the
  slice maximum when it is finite (else by 0), ``log(sum(exp(z - shift))) +
  shift``; an all ``-inf`` slice gives ``-inf``.
* ``PointCloudOracle``     -- PointCloudGeometry, sqeucl cost
  (geometry.py:214-354): cost block ``|x|^2 + |y|^2 - 2 x y^T`` clamped at 0
  (263-276), exact-zero diagonal for identical point sets (259-261,
  278-292), 256-row / 256-column streamed ``apply_lse_kernel`` (336-354),
  1000-pair ``mean_cost`` with ``default_rng(0)`` (294-312).
* ``DenseOracle``          -- DenseGeometry.apply_lse_kernel (geometry.py:204-211).
* ``EpsilonScheduleOracle`` -- EpsilonSchedule (geometry.py:75-97).
* ``as_weights``           -- sinkhorn._as_weights (sinkhorn.py:35-45).
* ``sinkhorn``             -- sinkhorn._sinkhorn_iterations (sinkhorn.py:151-200).
* ``dual_objective``       -- sinkhorn._dual_objective (sinkhorn.py:115-119).
* ``reg_ot_cost``          -- sinkhorn.reg_ot_cost (sinkhorn.py:210-216), row
  blocked so it never materialises the n x m plan (same sums, blocked order).
* ``transport_matrix``     -- sinkhorn.transport_matrix (sinkhorn.py:203-207).

Nothing in the product package imports this module.
"""

from __future__ import annotations

import numpy as np

BLOCK = 256          # geometry.py:44 DEFAULT_BLOCK_SIZE
MEAN_COST_SAMPLES = 1000   # geometry.py:42


class OracleValueError(ValueError):
    pass


def logsumexp(z: np.ndarray, axis: int) -> np.ndarray:
    """Max-shifted log-sum-exp (scipy.special.logsumexp semantics)."""
    z = np.asarray(z, dtype=np.float64)
    top = np.max(z, axis=axis, keepdims=True)
    shift = np.where(np.isfinite(top), top, 0.0)
    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        total = np.sum(np.exp(z - shift), axis=axis, keepdims=True)
        out = np.log(total) + shift
    return np.squeeze(out, axis=axis)


def _potential(p, size, name):
    # geometry.py:65-72: -inf allowed, NaN / +inf rejected.
    p = np.asarray(p, dtype=np.float64)
    if p.shape != (size,):
        raise OracleValueError(f"{name} must have shape ({size},), got {p.shape}")
    if np.isnan(p).any() or np.any(p == np.inf):
        raise OracleValueError(f"{name} contains NaN or +inf entries")
    return p


class EpsilonScheduleOracle:
    """eps_t = max(target, target * init_scale * decay**t) (geometry.py:96-97)."""

    def __init__(self, target, init_scale=1.0, decay=1.0):
        self.target = float(target)
        self.init_scale = float(init_scale)
        self.decay = float(decay)

    def at(self, t):
        return max(self.target, self.target * self.init_scale * self.decay ** t)


class PointCloudOracle:
    """Streamed point-cloud geometry in float64: sqeucl (default), eucl, cosine
    (geometry.py:263-276)."""

    def __init__(self, x, y, block_size=BLOCK, cost_fn="sqeucl"):
        if cost_fn not in ("sqeucl", "eucl", "cosine"):
            raise OracleValueError(f"unknown cost_fn {cost_fn!r}")
        self.cost_fn = cost_fn
        self.x = np.asarray(x, dtype=np.float64)
        self.y = np.asarray(y, dtype=np.float64)
        self.shape = (self.x.shape[0], self.y.shape[0])
        self.block_size = int(block_size)
        self.same_points = self.x is self.y or (
            self.x.shape == self.y.shape and np.array_equal(self.x, self.y))

    # --- cost blocks (geometry.py:263-292) ---
    def _sq_block(self, xs, ys):
        if self.cost_fn == "cosine":
            xn = xs / np.linalg.norm(xs, axis=1, keepdims=True)
            yn = ys / np.linalg.norm(ys, axis=1, keepdims=True)
            return 1.0 - xn @ yn.T
        nx = np.einsum("id,id->i", xs, xs)
        ny = np.einsum("jd,jd->j", ys, ys)
        blk = nx[:, None] + ny[None, :] - 2.0 * (xs @ ys.T)
        np.maximum(blk, 0.0, out=blk)
        if self.cost_fn == "eucl":
            return np.sqrt(blk)
        return blk

    def cost_rows(self, lo, hi):
        blk = self._sq_block(self.x[lo:hi], self.y)
        if self.same_points:
            k = np.arange(lo, min(hi, self.shape[1]))
            blk[k - lo, k] = 0.0
        return blk

    def cost_cols(self, lo, hi):
        blk = self._sq_block(self.x, self.y[lo:hi])
        if self.same_points:
            k = np.arange(lo, min(hi, self.shape[0]))
            blk[k, k - lo] = 0.0
        return blk

    def cost_matrix(self):
        return self.cost_rows(0, self.shape[0])

    def mean_cost(self):
        """Subsampled mean (geometry.py:294-312); exact when n*m <= 1000."""
        n, m = self.shape
        if n * m <= MEAN_COST_SAMPLES:
            return float(self.cost_matrix().mean())
        rng = np.random.default_rng(0)
        i = rng.integers(0, n, size=MEAN_COST_SAMPLES)
        j = rng.integers(0, m, size=MEAN_COST_SAMPLES)
        if self.cost_fn == "cosine":
            xn = self.x[i] / np.linalg.norm(self.x[i], axis=1, keepdims=True)
            yn = self.y[j] / np.linalg.norm(self.y[j], axis=1, keepdims=True)
            vals = 1.0 - np.einsum("kd,kd->k", xn, yn)
        else:
            diff = self.x[i] - self.y[j]
            vals = np.maximum(np.einsum("kd,kd->k", diff, diff), 0.0)
            if self.cost_fn == "eucl":
                vals = np.sqrt(vals)
        if self.same_points:
            vals = np.where(i == j, 0.0, vals)
        return float(vals.mean())

    # --- log-domain kernel (geometry.py:336-354) ---
    def apply_lse_kernel(self, f, g, eps, axis):
        n, m = self.shape
        f = _potential(f, n, "f")
        g = _potential(g, m, "g")
        bs = self.block_size
        if axis == "rows":
            out = np.empty(n)
            for lo in range(0, n, bs):
                hi = min(lo + bs, n)
                z = (f[lo:hi, None] + g[None, :] - self.cost_rows(lo, hi)) / eps
                out[lo:hi] = eps * logsumexp(z, axis=1)
            return out
        if axis != "cols":
            raise OracleValueError("axis must be 'rows' or 'cols'")
        out = np.empty(m)
        for lo in range(0, m, bs):
            hi = min(lo + bs, m)
            z = (f[:, None] + g[None, lo:hi] - self.cost_cols(lo, hi)) / eps
            out[lo:hi] = eps * logsumexp(z, axis=0)
        return out

    def rows_lse_subset(self, rows, g, eps):
        """eps*LSE_j((g_j - C_ij)/eps) for an arbitrary subset of rows.

        Each output reduces over its full axis in one call, so a subset gives
        exactly the reference values for those rows (geometry.py:220-223).
        """
        rows = np.asarray(rows)
        g = _potential(g, self.shape[1], "g")
        out = np.empty(rows.size)
        for lo in range(0, rows.size, self.block_size):
            sel = rows[lo:lo + self.block_size]
            blk = self._sq_block(self.x[sel], self.y)
            if self.same_points:
                hit = sel < self.shape[1]
                blk[np.nonzero(hit)[0], sel[hit]] = 0.0
            out[lo:lo + sel.size] = eps * logsumexp((g[None, :] - blk) / eps, axis=1)
        return out

    def cols_lse_subset(self, cols, f, eps):
        cols = np.asarray(cols)
        f = _potential(f, self.shape[0], "f")
        out = np.empty(cols.size)
        for lo in range(0, cols.size, self.block_size):
            sel = cols[lo:lo + self.block_size]
            blk = self._sq_block(self.x, self.y[sel])
            if self.same_points:
                hit = sel < self.shape[0]
                blk[sel[hit], np.nonzero(hit)[0]] = 0.0
            out[lo:lo + sel.size] = eps * logsumexp((f[:, None] - blk) / eps, axis=0)
        return out

    def row_blocks(self):
        for lo in range(0, self.shape[0], self.block_size):
            hi = min(lo + self.block_size, self.shape[0])
            yield lo, hi, self.cost_rows(lo, hi)


class DenseOracle:
    """Explicit cost matrix (geometry.py:171-211)."""

    def __init__(self, cost):
        self.cost = np.asarray(cost, dtype=np.float64)
        self.shape = self.cost.shape

    def cost_matrix(self):
        return self.cost

    def mean_cost(self):
        return float(self.cost.mean())

    def apply_lse_kernel(self, f, g, eps, axis):
        n, m = self.shape
        f = _potential(f, n, "f")
        g = _potential(g, m, "g")
        z = (f[:, None] + g[None, :] - self.cost) / eps
        return eps * logsumexp(z, axis=1 if axis == "rows" else 0)

    def row_blocks(self):
        for lo in range(0, self.shape[0], BLOCK):
            hi = min(lo + BLOCK, self.shape[0])
            yield lo, hi, self.cost[lo:hi]


def as_weights(w, size, name="w"):
    """sinkhorn.py:35-45: uniform default; shape, finite, >= 0, |sum-1| <= 1e-8."""
    if w is None:
        return np.full(size, 1.0 / size)
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (size,):
        raise OracleValueError(f"{name} must have shape ({size},)")
    if not np.all(np.isfinite(w)) or np.any(w < 0):
        raise OracleValueError(f"{name} must be entrywise finite and nonnegative")
    if abs(w.sum() - 1.0) > 1e-8:
        raise OracleValueError(f"{name} must sum to 1")
    return w


def dual_objective(f, g, a, b, eps, total_mass):
    """sinkhorn.py:115-119."""
    with np.errstate(invalid="ignore"):
        fa = np.where(a > 0, f * a, 0.0).sum()
        gb = np.where(b > 0, g * b, 0.0).sum()
    return float(fa + gb - eps * (total_mass - 1.0))


class OracleDiverged(Exception):
    def __init__(self, iteration):
        super().__init__(f"NaN in potentials (iteration {iteration})")
        self.iteration = iteration


def sinkhorn(geom, a, b, eps, threshold=1e-3, max_iters=2000, inner_iters=10,
             g_init=None):
    """Log-domain Sinkhorn loop (sinkhorn.py:151-200).

    ``eps`` is a float or an ``EpsilonScheduleOracle``.  Returns a dict with
    f, g, errors, dual_trace, iterations, converged, eps.
    """
    n, m = geom.shape
    a = as_weights(a, n, "a")
    b = as_weights(b, m, "b")
    sched = eps if isinstance(eps, EpsilonScheduleOracle) else EpsilonScheduleOracle(float(eps))
    target = sched.target
    with np.errstate(divide="ignore"):
        la = np.log(a)
        lb = np.log(b)
    zn, zm = np.zeros(n), np.zeros(m)
    f = np.zeros(n)
    g = np.zeros(m) if g_init is None else np.array(g_init, dtype=np.float64)
    errors, duals = [], []
    converged = False
    t = 0
    for t in range(1, max_iters + 1):
        e = sched.at(t - 1)
        f = e * la - geom.apply_lse_kernel(zn, g, e, "rows")
        g = e * lb - geom.apply_lse_kernel(f, zm, e, "cols")
        if t % inner_iters == 0 or t == max_iters:
            if np.isnan(f).any() or np.isnan(g).any():
                raise OracleDiverged(t)
            if e > target:
                continue
            row = np.exp(geom.apply_lse_kernel(f, g, e, "rows") / e)
            err = float(np.abs(row - a).sum())
            errors.append(err)
            duals.append(dual_objective(f, g, a, b, e, row.sum()))
            if err <= threshold:
                converged = True
                break
    return dict(f=f, g=g, errors=np.asarray(errors), dual_trace=np.asarray(duals),
                iterations=t, converged=converged, eps=target)


def marginal_check(geom, f, g, a, b, eps):
    """One check pass at given potentials (sinkhorn.py:183-186): (err, dual)."""
    row = np.exp(geom.apply_lse_kernel(f, g, eps, "rows") / eps)
    return float(np.abs(row - a).sum()), dual_objective(f, g, a, b, eps, row.sum())


def reg_ot_cost(geom, f, g, a, b, eps):
    """sinkhorn.py:210-216 without materialising: per row block, plan, sum C*P, sum P."""
    transport = 0.0
    mass = 0.0
    for lo, hi, cblk in geom.row_blocks():
        plan = np.exp((f[lo:hi, None] + g[None, :] - cblk) / eps)
        transport += float((cblk * plan).sum())
        mass += float(plan.sum())
    return transport, dual_objective(f, g, a, b, eps, mass)


def transport_matrix(geom, f, g, eps):
    """sinkhorn.py:203-207."""
    return np.exp((f[:, None] + g[None, :] - geom.cost_matrix()) / eps)
