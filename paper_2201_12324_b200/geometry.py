"""Cost geometries backed by the sm_100a library (drop-in for reference geometry.py).

Mirrors the reference's Geometry plugin API (geometry.py:100-168): solvers
only touch ``shape``, ``epsilon_default``, ``apply_lse_kernel`` and
``cost_matrix``.  Points, potentials and costs live on the GPU in float32;
inputs may be numpy arrays (results come back as float64 numpy, like the
reference) or CUDA torch tensors (results stay on the device).

Implemented: ``PointCloudGeometry`` with the squared-Euclidean cost (never
materialised: the online kernels of csrc/lse_simt.cu and csrc/lse_tc.cu), the
Euclidean cost (the same kernels with a square root per cell, OTK_COST_EUCL)
and the cosine cost (1 - <x^,y^> = |x^/sqrt2 - y^/sqrt2|^2: the sqeucl kernels
on normalised, 1/sqrt(2)-scaled points), ``DenseGeometry`` (stored cost,
csrc/dense.cu), ``EpsilonSchedule`` and the non-log ``apply_kernel`` (built on
the log-domain kernels).  Out of scope: ``GridGeometry``.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from ._device import (as_device_f32, device, is_torch, stream, to_output, validate_potential)

__all__ = [
    "Geometry",
    "DenseGeometry",
    "PointCloudGeometry",
    "EpsilonSchedule",
    "DEFAULT_EPSILON_SCALE",
    "DEFAULT_BLOCK_SIZE",
    "DEFAULT_DENSE_CAP",
    "COST_FNS",
]

DEFAULT_EPSILON_SCALE = 0.05        # geometry.py:40
_MEAN_COST_SAMPLES = 1000           # geometry.py:42
DEFAULT_BLOCK_SIZE = 256            # geometry.py:44 (accepted, performance-only)
DEFAULT_DENSE_CAP = 4_000_000       # geometry.py:46
COST_FNS = ("sqeucl", "eucl", "cosine")  # geometry.py:35
_REFERENCE_COST_FNS = ("sqeucl", "eucl", "cosine")
_LOG2E = 1.4426950408889634


def _check_axis(axis: str) -> None:
    if axis not in ("rows", "cols"):
        raise ValueError(f"axis must be 'rows' or 'cols', got {axis!r}")


class EpsilonSchedule:
    """Geometric decay toward a target: eps_t = max(target, target*init_scale*decay**t).

    Same parameters and validation as the reference (geometry.py:75-97).
    """

    def __init__(self, target: float, init_scale: float = 1.0, decay: float = 1.0):
        if not (target > 0):
            raise ValueError("target must be positive")
        if init_scale < 1.0:
            raise ValueError("init_scale must be >= 1")
        if not (0.0 < decay <= 1.0):
            raise ValueError("decay must lie in (0, 1]")
        if init_scale > 1.0 and decay == 1.0:
            raise ValueError("schedule with init_scale > 1 and decay = 1 never reaches its target")
        self.target = float(target)
        self.init_scale = float(init_scale)
        self.decay = float(decay)

    def at(self, t: int) -> float:
        return max(self.target, self.target * self.init_scale * self.decay ** t)


class Geometry:
    """Abstract cost structure between n source and m target locations."""

    _shape: tuple[int, int]
    _epsilon_default: float | None

    @property
    def shape(self) -> tuple[int, int]:
        return self._shape

    @property
    def epsilon_default(self) -> float:
        if self._epsilon_default is None:
            self._epsilon_default = DEFAULT_EPSILON_SCALE * self.mean_cost()
        return self._epsilon_default

    def mean_cost(self) -> float:
        raise NotImplementedError

    def cost_matrix(self, max_entries: int | None = None):
        raise NotImplementedError

    def apply_kernel(self, v, eps=None, axis="rows"):
        """K v (rows) or K^T v (cols) with K = exp(-C/eps) (geometry.py:130-139).

        Built on the log-domain kernel: with v = v+ - v-,
        K v+ = exp(LSE_j(log v+_j - C_ij/eps)) = exp(apply_lse_kernel(0, eps log v+)/eps),
        one device half-step per sign present.  float32 device arithmetic: the
        result carries ~1e-6 relative error per part, and heavy cancellation
        between the parts loses accuracy the float64 reference keeps.
        """
        _check_axis(axis)
        eps = self._resolve_eps(eps)
        n, m = self.shape
        size, out_size = (m, n) if axis == "rows" else (n, m)
        like = v
        if is_torch(v):
            v = v.detach().double().cpu().numpy()
        v = np.asarray(v, dtype=float)
        if v.shape != (size,):
            raise ValueError(f"v must have shape ({size},), got {v.shape}")
        if not np.all(np.isfinite(v)):
            raise ValueError("v contains non-finite entries")
        out = np.zeros(out_size)
        for sign, part in ((1.0, np.maximum(v, 0.0)), (-1.0, np.maximum(-v, 0.0))):
            if not np.any(part > 0):
                continue
            with np.errstate(divide="ignore"):
                pot = eps * np.log(part)
            zeros = np.zeros(out_size)
            f, g = (zeros, pot) if axis == "rows" else (pot, zeros)
            lse = np.asarray(self.apply_lse_kernel(f, g, eps, axis), dtype=float)
            with np.errstate(over="ignore"):
                out += sign * np.exp(lse / eps)
        if is_torch(like):
            import torch
            return torch.as_tensor(out, dtype=torch.float32, device=device())
        return out

    def apply_lse_kernel(self, f, g, eps=None, axis="rows"):
        raise NotImplementedError

    def _resolve_eps(self, eps) -> float:
        if eps is None:
            return self.epsilon_default
        eps = float(eps)
        if not (eps > 0):
            raise ValueError("eps must be positive")
        return eps

    def _check_cap(self, max_entries: int | None) -> None:
        # Reads the module global at call time, like the reference (geometry.py:162-168).
        cap = DEFAULT_DENSE_CAP if max_entries is None else int(max_entries)
        n, m = self.shape
        if n * m > cap:
            raise ValueError(
                f"cost matrix with {n}x{m} = {n * m} entries exceeds the materialization cap {cap}")


def _validate_points(p, name):
    if is_torch(p):
        if p.ndim != 2:
            raise ValueError("x and y must be 2-D arrays of shape (num_points, dim)")
        if p.shape[0] == 0:
            raise ValueError("point sets must be non-empty")
        return p
    p = np.asarray(p, dtype=float)
    if p.ndim != 2:
        raise ValueError("x and y must be 2-D arrays of shape (num_points, dim)")
    if p.shape[0] == 0:
        raise ValueError("point sets must be non-empty")
    return p


def _cuda_available() -> bool:
    import torch
    return torch.cuda.is_available()


def _has_zero_row(p) -> bool:
    if is_torch(p):
        import torch
        return bool((torch.linalg.vector_norm(p.double(), dim=1) == 0).any().item())
    return bool(np.any(np.linalg.norm(p, axis=1) == 0))


def _all_finite(p) -> bool:
    if is_torch(p):
        import torch
        return bool(torch.isfinite(p).all().item())
    return bool(np.all(np.isfinite(p)))


class _Cloud:
    """Device-resident point set: fp32 points, squared norms and, on the tcgen05 path (every d),
    the split-fp16 operand planes (hi, lo) and norm planes (ext_a, ext_b) of
    the tcgen05 kernel, all scaled by the geometry's common power-of-two s."""

    def __init__(self, pts):
        import torch
        self.p = as_device_f32(pts).contiguous()
        self.n, self.d = self.p.shape
        self.sq = torch.empty(self.n, dtype=torch.float32, device=self.p.device)
        self.dpad = (self.d + 63) // 64 * 64
        self.hi = self.lo = self.ext_a = self.ext_b = None
        self.scale = 1.0

    def absmax(self) -> float:
        import torch
        amax = torch.empty(1, dtype=torch.float32, device=self.p.device)
        N.check(N.lib().otk_absmax(N.ptr(self.p), self.n * self.d, N.ptr(amax), stream()), "absmax")
        return float(amax.item())

    def prepare(self, scale: float, planes: bool):
        import torch
        self.scale = float(scale)
        if planes:
            dev = self.p.device
            self.hi = torch.empty((self.n, self.dpad), dtype=torch.float16, device=dev)
            self.lo = torch.empty_like(self.hi)
            self.ext_a = torch.empty((self.n, 16), dtype=torch.float16, device=dev)
            self.ext_b = torch.empty_like(self.ext_a)
        N.check(N.lib().otk_prep_points(N.ptr(self.p), self.n, self.d, N.ptr(self.sq),
                                        N.ptr(self.hi), N.ptr(self.lo), N.ptr(self.ext_a),
                                        N.ptr(self.ext_b), self.dpad, self.scale, stream()), "prep")
        return self


def kernel_points(p, cost_fn: str):
    """Points the kernels see: cosine -> x/|x|/sqrt(2) (float64 math), so that
    |x'-y'|^2 = 1 - <x^, y^> (geometry.py:264-267); sqeucl / eucl -> x."""
    if cost_fn != "cosine":
        return p
    if is_torch(p):
        q = as_device_f32(p).double()
        return (q / q.norm(dim=1, keepdim=True) / np.sqrt(2.0)).float().contiguous()
    q = np.asarray(p, dtype=np.float64)
    return q / np.linalg.norm(q, axis=1, keepdims=True) / np.sqrt(2.0)


def centered_points(px, py, cost_fn: str, same: bool = False):
    """The kernel points of both sets, shifted by one common centre (the
    coordinate-wise median of y; otk_column_median / otk_shift_points).  sqeucl and eucl
    costs are translation-invariant (geometry.py:268-275), and the float32
    norm form |x|^2 + |y|^2 - 2<x,y> the kernels use then loses precision only
    with the spread of the points, not with their offset from the origin.  y is
    replicated on every rank of a sharded solve, so every rank derives the same
    centre.  cosine points are normalised instead (kernel_points)."""
    import torch
    kx = as_device_f32(kernel_points(px, cost_fn)).contiguous()
    ky = kx if same else as_device_f32(kernel_points(py, cost_fn)).contiguous()
    if cost_fn == "cosine":
        return kx, ky
    lib = N.lib()
    m, d = ky.shape
    dev = ky.device
    center = torch.empty(d, dtype=torch.float64, device=dev)
    st = stream()
    N.check(lib.otk_column_median(N.ptr(ky), m, d, N.ptr(center), st), "column median")
    cy = torch.empty_like(ky)
    N.check(lib.otk_shift_points(N.ptr(ky), m, d, N.ptr(center), N.ptr(cy), st), "shift y")
    if same:
        return cy, cy
    cx = torch.empty_like(kx)
    N.check(lib.otk_shift_points(N.ptr(kx), kx.shape[0], d, N.ptr(center), N.ptr(cx), st), "shift x")
    return cx, cy


_PAIR_CACHE: dict = {}


def _mean_cost_pairs(n: int, m: int, dev):
    """The reference's seeded sample of index pairs (geometry.py:296-298:
    default_rng(0), i then j), as device int64 tensors; they depend only on the
    shape, so they are drawn and uploaded once per (n, m, device)."""
    import torch
    key = (n, m, str(dev))
    hit = _PAIR_CACHE.get(key)
    if hit is None:
        rng = np.random.default_rng(0)
        i = rng.integers(0, n, size=_MEAN_COST_SAMPLES)
        j = rng.integers(0, m, size=_MEAN_COST_SAMPLES)
        hit = (torch.as_tensor(i, dtype=torch.int64, device=dev), torch.as_tensor(j, dtype=torch.int64, device=dev))
        if len(_PAIR_CACHE) > 64:
            _PAIR_CACHE.clear()
        _PAIR_CACHE[key] = hit
    return hit


def cost_fn_flags(cost_fn: str) -> int:
    if cost_fn not in COST_FNS:
        raise ValueError(f"cost_fn must be one of {COST_FNS}, got {cost_fn!r}")
    return N.OTK_COST_EUCL if cost_fn == "eucl" else 0


class PointCloudGeometry(Geometry):
    """Squared-Euclidean costs between two point sets, never materialised.

    Same constructor and validation as the reference (geometry.py:226-261).
    ``block_size`` is accepted for API compatibility; like the reference it
    never changes results (the GPU kernels pick their own tiles).
    """

    def __init__(self, x, y, cost_fn: str = "sqeucl", epsilon_default: float | None = None,
                 block_size: int = DEFAULT_BLOCK_SIZE):
        same_obj = x is y
        x = _validate_points(x, "x")
        y = x if same_obj else _validate_points(y, "y")
        if x.shape[1] != y.shape[1]:
            raise ValueError(f"dimension mismatch: x has d={x.shape[1]}, y has d={y.shape[1]}")
        # torch inputs (host or device) are moved to the GPU once and validated
        # there; the device copies are the ones the kernels use (_clouds)
        self._dev_pts = None
        if (is_torch(x) or is_torch(y)) and _cuda_available():
            xd = as_device_f32(x, async_pinned=True)
            self._dev_pts = (xd, xd if same_obj else as_device_f32(y, async_pinned=True))
        vx, vy = self._dev_pts if self._dev_pts is not None else (x, y)
        same_dev = None
        if self._dev_pts is not None:
            # one launch and one device->host read for both finiteness flags and the
            # same-points test (otk_points_flags)
            import torch
            compare = (not same_obj) and tuple(x.shape) == tuple(y.shape)
            fl = torch.empty(3, dtype=torch.int32, device=vx.device)
            N.check(N.lib().otk_points_flags(N.ptr(vx), vx.shape[0], N.ptr(vy), vy.shape[0],
                                             int(vx.shape[1]), 1 if compare else 0, N.ptr(fl), stream()),
                    "points flags")
            got = fl.cpu().tolist()
            finite = got[0] == 0 and got[1] == 0
            same_dev = compare and got[2] == 0
        else:
            finite = _all_finite(vx) and (same_obj or _all_finite(vy))
        if not finite:
            raise ValueError("points contain non-finite entries")
        if cost_fn not in _REFERENCE_COST_FNS:
            raise ValueError(f"cost_fn must be one of {_REFERENCE_COST_FNS}, got {cost_fn!r}")
        if cost_fn == "cosine" and (_has_zero_row(vx) or (not same_obj and _has_zero_row(vy))):
            raise ValueError("cosine cost is undefined for zero vectors")
        if epsilon_default is not None and not (epsilon_default > 0):
            raise ValueError("epsilon_default must be positive")
        if block_size < 1:
            raise ValueError("block_size must be >= 1")
        self.x = x
        self.y = y
        self.cost_fn = cost_fn
        self.block_size = int(block_size)
        self._shape = (int(x.shape[0]), int(y.shape[0]))
        self._epsilon_default = epsilon_default
        if same_obj:
            self._same_points = True
        elif self._dev_pts is not None:
            self._same_points = same_dev
        else:
            self._same_points = bool(x.shape == y.shape and np.array_equal(x, y))
        self._dev = None
        self._kpts = None
        self.impl_flags = 0  # N.OTK_IMPL_SIMT / N.OTK_IMPL_TC to force a kernel

    # ---- device state (lazy: construction and validation need no GPU)
    def _kernel_points(self, p):
        return kernel_points(p, self.cost_fn)

    def _points(self):
        """fp32 device points the kernels see (cosine: normalised; sqeucl / eucl:
        centred on the coordinate-wise median of y, centered_points), cached; the whole-solve
        entry needs only these (it prepares norms / planes itself)."""
        if self._kpts is None:
            device()
            px, py = self._dev_pts if self._dev_pts is not None else (self.x, self.y)
            self._kpts = centered_points(px, py, self.cost_fn, same=self._same_points)
        return self._kpts

    def _clouds(self):
        if self._dev is None:
            kx, ky = self._points()
            cx = _Cloud(kx)
            cy = cx if self._same_points else _Cloud(ky)
            planes = bool(N.lib().otk_lse_uses_tc(cx.d, self.impl_flags))
            scale = 1.0
            if planes:
                amax = max(cx.absmax(), cy.absmax())
                scale = float(N.lib().otk_split_scale(amax, cx.d))
            cx.prepare(scale, planes)
            if cy is not cx:
                cy.prepare(scale, planes)
            self._dev = (cx, cy)
        return self._dev

    @property
    def _cost_flags(self):
        """OTK_SAME_POINTS / OTK_COST_EUCL for every kernel that forms a cost."""
        return ((N.OTK_SAME_POINTS if self._same_points else 0) |
                (N.OTK_COST_EUCL if self.cost_fn == "eucl" else 0))

    @property
    def _flags(self):
        return N.OTK_CLAMP | self._cost_flags | self.impl_flags

    def mean_cost(self) -> float:
        """0.05 * this is epsilon_default; subsampled like geometry.py:294-312."""
        import torch
        n, m = self.shape
        if n * m <= _MEAN_COST_SAMPLES:
            return float(torch.as_tensor(self.cost_matrix(max_entries=n * m)).mean())
        # the kernel points are enough (no norms / operand planes); cosine: they are
        # x^/sqrt2, so |x'-y'|^2 = 1 - <x^,y^> (geometry.py:303-306)
        kx, ky = self._points()
        ii, jj = _mean_cost_pairs(n, m, kx.device)
        out = torch.empty(1, dtype=torch.float64, device=kx.device)
        N.check(N.lib().otk_mean_cost_pairs(N.ptr(kx), N.ptr(ky), N.ptr(ii), N.ptr(jj), ii.numel(),
                                            int(kx.shape[1]), self._cost_flags, N.ptr(out), stream()),
                "mean cost")
        return float(out.item())

    def cost_matrix(self, max_entries: int | None = None):
        """Materialise C on the GPU (difference form); refuses past the cap."""
        import torch
        self._check_cap(max_entries)
        cx, cy = self._clouds()
        n, m = self.shape
        out = torch.empty((n, m), dtype=torch.float32, device=cx.p.device)
        N.check(N.lib().otk_dense_cost(N.ptr(cx.p), N.ptr(cy.p), 1, n, m, cx.d,
                                       self._cost_flags, N.ptr(out),
                                       None, stream()), "cost_matrix")
        return to_output(out, self.x)

    def apply_lse_kernel(self, f, g, eps=None, axis="rows"):
        """rows: f_i + eps*LSE_j((g_j - C_ij)/eps); cols: the same over i (geometry.py:336-354)."""
        import torch
        _check_axis(axis)
        eps = self._resolve_eps(eps)
        n, m = self.shape
        like = f
        f = validate_potential(f, n, "f")
        g = validate_potential(g, m, "g")
        cx, cy = self._clouds()
        kappa = float(np.float32(_LOG2E / eps))
        if axis == "rows":
            P, Q, base, qpot, npts, nq = cx, cy, f, g, n, m
        else:
            P, Q, base, qpot, npts, nq = cy, cx, g, f, m, n
        lib = N.lib()
        st = stream()
        bias = torch.empty(nq, dtype=torch.float32, device=cx.p.device)
        N.check(lib.otk_make_bias(N.ptr(qpot), nq, kappa, N.ptr(bias), None, 0, st))
        flags = self._flags
        nsplit = lib.otk_lse_suggest_nsplit(npts, nq, cx.d, flags)
        part = torch.empty(nsplit * npts, dtype=torch.float32, device=cx.p.device)
        sinv = 1.0 / (cx.scale * cx.scale)
        N.check(lib.otk_lse_partial(N.ptr(P.p), N.ptr(P.sq), N.ptr(P.hi), N.ptr(P.lo),
                                    N.ptr(P.ext_a), npts, N.ptr(Q.p), N.ptr(Q.sq), N.ptr(Q.hi),
                                    N.ptr(Q.lo), N.ptr(Q.ext_b), nq, cx.d, cx.dpad, sinv,
                                    N.ptr(bias), kappa, flags, nsplit, N.ptr(part), st),
                "apply_lse_kernel")
        out = torch.empty(npts, dtype=torch.float32, device=cx.p.device)
        N.check(lib.otk_lse_finalize(N.ptr(part), nsplit, npts, N.ptr(base), N.OTK_FIN_APPLY,
                                     float(eps), 0.0, N.ptr(out), None, None, 0, st), "finalize")
        return to_output(out, like)


class DenseGeometry(Geometry):
    """Geometry backed by an explicit cost matrix (geometry.py:171-211), stored on the GPU."""

    def __init__(self, cost, epsilon_default: float | None = None):
        if is_torch(cost):
            if cost.ndim != 2 or cost.numel() == 0:
                raise ValueError(f"cost must be a non-empty 2-D array, got shape {tuple(cost.shape)}")
        else:
            cost = np.asarray(cost, dtype=float)
            if cost.ndim != 2 or cost.size == 0:
                raise ValueError(f"cost must be a non-empty 2-D array, got shape {cost.shape}")
        if not _all_finite(cost):
            raise ValueError("cost matrix contains non-finite entries")
        if epsilon_default is not None and not (epsilon_default > 0):
            raise ValueError("epsilon_default must be positive")
        self._cost_in = cost
        self._shape = (int(cost.shape[0]), int(cost.shape[1]))
        self._epsilon_default = epsilon_default
        self._dev = None

    def _c(self):
        if self._dev is None:
            device()
            self._dev = as_device_f32(self._cost_in).contiguous()
        return self._dev

    def _c_ct(self):
        """(C, C^T) on the device; C^T lets the column half-steps stream row-major."""
        import torch
        C = self._c()
        if getattr(self, "_ct", None) is None:
            n, m = self.shape
            ct = torch.empty((m, n), dtype=torch.float32, device=C.device)
            N.check(N.lib().otk_dense_transpose(N.ptr(C), 1, n, m, N.ptr(ct), stream()),
                    "dense_transpose")
            self._ct = ct
        return C, self._ct

    def mean_cost(self) -> float:
        if is_torch(self._cost_in):
            return float(self._cost_in.double().mean().item())
        return float(self._cost_in.mean())

    def cost_matrix(self, max_entries: int | None = None):
        self._check_cap(max_entries)
        return self._cost_in

    def apply_lse_kernel(self, f, g, eps=None, axis="rows"):
        import torch
        _check_axis(axis)
        eps = self._resolve_eps(eps)
        n, m = self.shape
        like = f
        f = validate_potential(f, n, "f")
        g = validate_potential(g, m, "g")
        C = self._c()
        kappa = float(np.float32(_LOG2E / eps))
        if axis == "rows":
            qpot, base, nout, nq = g, f, n, m
        else:
            qpot, base, nout, nq = f, g, m, n
        in_bias = torch.empty(nq, dtype=torch.float32, device=C.device)
        N.check(N.lib().otk_make_bias(N.ptr(qpot), nq, kappa, N.ptr(in_bias), None, 0, stream()))
        eps_t = torch.tensor([eps], dtype=torch.float32, device=C.device)
        out = torch.empty(nout, dtype=torch.float32, device=C.device)
        N.check(N.lib().otk_dense_lse(N.ptr(C), 1, n, m, 0 if axis == "rows" else 1,
                                      N.ptr(in_bias), N.ptr(base), N.OTK_FIN_APPLY,
                                      N.ptr(eps_t), None, None, N.ptr(out), None, None, 0,
                                      stream()), "apply_lse_kernel")
        return to_output(out, like)
