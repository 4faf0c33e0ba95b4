"""Log-domain Sinkhorn on the GPU (drop-in for reference sinkhorn.py).

Same names, signatures, defaults, validation and exceptions as the
reference (sinkhorn.py:1-246) for the point-cloud / dense linear problem:

* ``solve_sinkhorn`` on a ``PointCloudGeometry`` runs the whole loop natively
  (``otk_solve_pointcloud``: online tcgen05 / FP32 half-steps, fused check,
  CUDA graphs); on a ``DenseGeometry`` it runs the materialised-cost kernels.
* ``reg_ot_cost`` is computed online (no n x m materialisation, so the
  reference's 4e6-entry cap does not apply); ``transport_matrix`` keeps the cap.
* ``solve_sinkhorn_batched`` (extension, no reference equivalent) solves B
  independent materialised problems in lock-step; each result equals an
  independent ``solve_sinkhorn`` call, iteration count included.

Outputs: ``SinkhornOutput.f``/``g`` are float64 numpy arrays like the
reference; ``f_device``/``g_device`` hold the float32 CUDA tensors.
"""

from __future__ import annotations

import dataclasses
import threading
import logging
from typing import NamedTuple

import ctypes
import os
from collections.abc import Sequence

import numpy as np

from . import _native as N
from ._device import as_device_f32, device, is_torch, nvtx_range, stream, to_output
from .errors import DivergedError
from .geometry import DenseGeometry, EpsilonSchedule, Geometry, PointCloudGeometry

logger = logging.getLogger(__name__)

__all__ = [
    "LinearProblem",
    "SinkhornOutput",
    "Coupling",
    "RegOTCost",
    "solve_sinkhorn",
    "solve_sinkhorn_batched",
    "BatchedSinkhornOutput",
    "transport_matrix",
    "reg_ot_cost",
    "grad_weights",
    "grad_points",
]

_LOG2E = 1.4426950408889634
_FLT_MIN = 1.1754943508222875e-38


def _as_weights(w, size: int, name: str) -> np.ndarray:
    """sinkhorn.py:35-45."""
    if w is None:
        return np.full(size, 1.0 / size)
    if is_torch(w):
        w = w.detach().double().cpu().numpy()
    w = np.asarray(w, dtype=float)
    if w.shape != (size,):
        raise ValueError(f"{name} must have shape ({size},), got {w.shape}")
    if not np.all(np.isfinite(w)) or np.any(w < 0):
        raise ValueError(f"{name} must be entrywise finite and nonnegative")
    if abs(w.sum() - 1.0) > 1e-8:
        raise ValueError(f"{name} must sum to 1, got {w.sum()!r}")
    return w


@dataclasses.dataclass(frozen=True, eq=False)
class LinearProblem:
    """A geometry plus two marginal histograms (uniform by default)."""

    geom: Geometry
    a: np.ndarray | None = None
    b: np.ndarray | None = None

    def __post_init__(self):
        n, m = self.geom.shape
        object.__setattr__(self, "a", _as_weights(self.a, n, "a"))
        object.__setattr__(self, "b", _as_weights(self.b, m, "b"))
        object.__setattr__(self, "_dev", None)

    def _weights(self):
        """float32 device weights and log-weights (logs taken in float64)."""
        if self._dev is None:
            with np.errstate(divide="ignore"):
                la, lb = np.log(self.a), np.log(self.b)
            # one host->device copy for the four vectors
            n, m = self.a.shape[0], self.b.shape[0]
            packed = as_device_f32(np.concatenate([self.a, self.b, la, lb]))
            object.__setattr__(self, "_dev", (packed[:n], packed[n:n + m], packed[n + m:2 * n + m],
                                              packed[2 * n + m:]))
        return self._dev


@dataclasses.dataclass(frozen=True, eq=False)
class SinkhornOutput:
    f: np.ndarray
    g: np.ndarray
    errors: np.ndarray
    dual_trace: np.ndarray
    iterations: int
    converged: bool
    eps: float
    f_device: object = dataclasses.field(default=None, repr=False)
    g_device: object = dataclasses.field(default=None, repr=False)


class BatchedSinkhornOutput(Sequence):
    """The B results of ``solve_sinkhorn_batched`` (extension; no reference equivalent).

    A read-only sequence: element k is the ``SinkhornOutput`` an independent
    ``solve_sinkhorn`` call on problem k returns (built on first access).  The
    batched arrays are also exposed directly -- ``f`` [B,n], ``g`` [B,m]
    (float64), ``iterations``, ``converged``, ``eps`` ([B]) and the float32
    device tensors ``f_device`` / ``g_device`` -- so callers of big batches
    need not materialise B Python objects.
    """

    def __init__(self, f, g, err_tab, dual_tab, n_rec, iterations, converged, eps, f_device,
                 g_device):
        # f / g / the trace tables may be device tensors: copied to the host on
        # first access (a batch whose potentials stay on the GPU never pays it)
        self._f, self._g = f, g
        self._err_src, self._dual_src, self._n = err_tab, dual_tab, n_rec
        self.iterations, self.converged, self.eps = iterations, converged, eps
        self.f_device, self.g_device = f_device, g_device
        self._cache = {}

    @staticmethod
    def _host(v, dtype):
        return v if isinstance(v, np.ndarray) else v.cpu().numpy().astype(dtype)

    @property
    def f(self):
        self._f = self._host(self._f, np.float64)
        return self._f

    @property
    def g(self):
        self._g = self._host(self._g, np.float64)
        return self._g

    @property
    def _err(self):
        self._err_src = self._host(self._err_src, np.float64)
        return self._err_src

    @property
    def _dual(self):
        self._dual_src = self._host(self._dual_src, np.float64)
        return self._dual_src

    def __len__(self):
        return len(self.iterations)

    def _one(self, k):
        if k not in self._cache:
            nk = int(self._n[k])
            self._cache[k] = SinkhornOutput(
                f=self.f[k], g=self.g[k], errors=self._err[k, :nk].copy(),
                dual_trace=self._dual[k, :nk].copy(), iterations=int(self.iterations[k]),
                converged=bool(self.converged[k]), eps=float(self.eps[k]),
                f_device=self.f_device[k], g_device=self.g_device[k])
        return self._cache[k]

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self._one(i) for i in range(*k.indices(len(self)))]
        k = int(k)
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        return self._one(k)


@dataclasses.dataclass(frozen=True, eq=False)
class Coupling:
    """A transport plan, stored as its dense matrix."""

    matrix: np.ndarray

    def row_marginal(self) -> np.ndarray:
        return self.matrix.sum(axis=1)

    def col_marginal(self) -> np.ndarray:
        return self.matrix.sum(axis=0)


class RegOTCost(NamedTuple):
    transport_cost: float
    dual_objective: float


def _resolve_schedule(geom: Geometry, eps) -> EpsilonSchedule:
    """sinkhorn.py:104-112."""
    if eps is None:
        eps = geom.epsilon_default
    if isinstance(eps, EpsilonSchedule):
        return eps
    eps = float(eps)
    if not (eps > 0):
        raise ValueError("eps must be positive")
    return EpsilonSchedule(eps)


def _dual_objective(f, g, a, b, eps, total_mass):
    """sinkhorn.py:115-119."""
    with np.errstate(invalid="ignore"):
        fa = np.where(a > 0, f * a, 0.0).sum()
        gb = np.where(b > 0, g * b, 0.0).sum()
    return float(fa + gb - eps * (total_mass - 1.0))


def _fp32_guard(sched: EpsilonSchedule, inner_iters: int, max_iters: int) -> None:
    # The device path computes in float32: an eps below the float32 normal
    # range makes every potential NaN.  The reference (float64) detects that
    # NaN at its first check; we report it at the same place without running.
    if sched.target < _FLT_MIN or not np.isfinite(np.float32(_LOG2E / sched.target)):
        raise DivergedError(
            "NaN in Sinkhorn potentials; eps is likely too small for the cost scale "
            "(below the float32 range of the device solver)",
            iteration=min(inner_iters, max_iters))


def solve_sinkhorn(prob: LinearProblem, eps=None, *, threshold: float = 1e-3, max_iters: int = 2000,
                   inner_iters: int = 10, g_init=None, impl: str = "auto",
                   use_graphs: bool = True, fixed_iters: bool = False) -> SinkhornOutput:
    """Runs log-domain Sinkhorn iterations until the marginals match (sinkhorn.py:122-148).

    ``impl`` ("auto" | "simt" | "tc" | "tc-noanchor") and ``use_graphs`` are performance knobs
    that never change results beyond float32 rounding.  ``g_init`` is the
    warm start of the reference's internal ``_sinkhorn_iterations``.
    ``fixed_iters`` is a measurement knob: the checks run and are recorded but
    never stop the loop, so exactly ``max_iters`` iterations run (float32
    iterates can reach an exact fixed point -- marginal error 0.0 -- which
    satisfies any threshold, however small).
    """
    if max_iters < 1 or inner_iters < 1:
        raise ValueError("max_iters and inner_iters must be >= 1")
    if not (threshold > 0):
        raise ValueError("threshold must be positive")
    geom = prob.geom
    sched = _resolve_schedule(geom, eps)
    _fp32_guard(sched, inner_iters, max_iters)
    if fixed_iters:
        threshold = -1.0  # err <= threshold never holds (the native loops accept a negative threshold)
    if isinstance(geom, PointCloudGeometry):
        return _solve_pointcloud(prob, sched, threshold, max_iters, inner_iters, g_init, impl,
                                 use_graphs)
    if isinstance(geom, DenseGeometry):
        C, CT = geom._c_ct()
        outs = _dense_loop(C[None], CT[None], prob._weights(), [sched], threshold, max_iters,
                           inner_iters, g_init=g_init)
        return outs[0]
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def _impl_flags(impl: str) -> int:
    if impl == "auto":
        return 0
    if impl == "simt":
        return N.OTK_IMPL_SIMT
    if impl == "tc":
        return N.OTK_IMPL_TC
    if impl == "tc-noanchor":  # A/B knob: running-max half-steps only
        return N.OTK_IMPL_TC | N.OTK_IMPL_NOANCHOR
    raise ValueError("impl must be 'auto', 'simt', 'tc' or 'tc-noanchor'")


def _raise_status(rc: int, iteration: int):
    if rc == N.OTK_DIVERGED:
        raise DivergedError(
            "NaN in Sinkhorn potentials; eps is likely too small for the cost scale",
            iteration=iteration)
    if rc == N.OTK_BAD_POTENTIAL:
        raise ValueError(f"g contains NaN or +inf entries (potential fed to iteration {iteration})")
    N.check(rc, "solve_sinkhorn")


_GEOM_LOCK = threading.Lock()


def _host_buffers(geom, n_pad: int, m: int, nbytes: int, dev):
    """Per-geometry reusable buffers of the whole-solve entry: the device
    workspace and a pinned host staging buffer for f | g (the solver copies
    the potentials there before its single final sync).  Reused by every
    solve on the geometry -- a solve's outputs are copied out of them."""
    import torch
    cache = getattr(geom, "_solve_bufs", None)
    if cache is None or cache["ws"].numel() < nbytes or cache["host"].numel() < n_pad + m \
            or cache["ws"].device != dev:
        cache = {"ws": torch.empty(nbytes, dtype=torch.uint8, device=dev),
                 "host": torch.empty(n_pad + m, dtype=torch.float32).pin_memory(),
                 "lock": cache["lock"] if cache else threading.Lock()}
        geom._solve_bufs = cache
    return cache


def _solve_pointcloud(prob, sched, threshold, max_iters, inner_iters, g_init, impl, use_graphs):
    import torch
    geom: PointCloudGeometry = prob.geom
    px, py = geom._points()  # the native solve prepares norms / operand planes itself
    a, b, la, lb = prob._weights()
    n, m = geom.shape
    d = int(px.shape[1])
    dev = px.device
    # f and g in one device buffer (the outputs' f_device / g_device); g starts
    # on a 256-byte boundary, as every separately allocated potential does
    n_pad = (n + 63) // 64 * 64
    fg = torch.empty(n_pad + m, dtype=torch.float32, device=dev)
    f_out, g_out = fg[:n], fg[n_pad:]
    max_checks = max_iters // inner_iters + 2
    errs = np.zeros(max_checks)
    duals = np.zeros(max_checks)
    gi = None
    if g_init is not None:
        gi = as_device_f32(g_init)
        if tuple(gi.shape) != (m,):
            raise ValueError(f"g_init must have shape ({m},)")
    A = N.SolveArgs()
    A.x, A.y, A.n, A.m, A.d = N.ptr(px), N.ptr(py), n, m, d
    A.a, A.b, A.log_a, A.log_b = N.ptr(a), N.ptr(b), N.ptr(la), N.ptr(lb)
    A.same_points = 1 if geom._same_points else 0
    A.eps_target, A.eps_init_scale, A.eps_decay = sched.target, sched.init_scale, sched.decay
    A.threshold, A.max_iters, A.inner_iters = float(threshold), int(max_iters), int(inner_iters)
    A.g_init = N.ptr(gi)
    A.flags = _impl_flags(impl) | geom.impl_flags | (geom._cost_flags & N.OTK_COST_EUCL)
    A.use_graphs = 1 if use_graphs else 0
    A.f_out, A.g_out = N.ptr(f_out), N.ptr(g_out)
    A.errors = errs.ctypes.data_as(ctypes.c_void_p)
    A.duals = duals.ctypes.data_as(ctypes.c_void_p)
    A.max_checks = max_checks
    lib = N.lib()
    nbytes = lib.otk_solve_workspace_bytes(ctypes.byref(A))
    with _GEOM_LOCK:
        bufs = _host_buffers(geom, n_pad, m, nbytes, dev)
    with bufs["lock"]:  # instances may be shared between threads (reference SPEC.md:94)
        host = bufs["host"]
        A.workspace, A.workspace_bytes, A.stream = N.ptr(bufs["ws"]), bufs["ws"].numel(), stream()
        A.f_host, A.g_host = host.data_ptr(), host.data_ptr() + 4 * n_pad
        rc = lib.otk_solve_pointcloud(ctypes.byref(A))
        if rc != N.OTK_OK:
            _raise_status(rc, A.fail_iter)
        fg_host = host.numpy()  # filled by the solver before its final sync
        f_h = fg_host[:n].astype(np.float64)
        g_h = fg_host[n_pad:n_pad + m].astype(np.float64)
    k = A.n_checks
    if not A.converged:
        logger.info("sinkhorn: no convergence after %d iterations (last error %s)", A.iterations,
                    errs[k - 1] if k else None)
    return SinkhornOutput(
        f=f_h, g=g_h, errors=errs[:k].copy(), dual_trace=duals[:k].copy(),
        iterations=int(A.iterations), converged=bool(A.converged), eps=sched.target,
        f_device=f_out, g_device=g_out)


# ---------------------------------------------------------------- dense / batched
def _dense_loop(C, CT, weights, scheds, threshold, max_iters, inner_iters, g_init=None,
                raise_on_fail=True):
    """Lock-step Sinkhorn over B stored-cost problems C[B,n,m] (csrc/dense.cu kernels).

    Each problem follows the reference loop (sinkhorn.py:151-200) exactly:
    its own eps schedule target, check cadence, NaN / bad-potential handling
    and convergence; converged problems are frozen (active mask).  Both
    half-steps stream their cost row-major: rows over C, columns over
    CT = C^T[B,m,n] (built once), so each is one coalesced HBM pass.
    weights = (a, b, log a, log b) as float32 CUDA tensors of shape [B,n] / [B,m]
    (or [n] / [m] when B == 1).  Per-problem bookkeeping at the checks is
    vectorised (numpy on the B check records; device index copies to freeze).
    """
    import torch
    lib = N.lib()
    st = stream()
    B, n, m = C.shape
    dev = C.device
    a, b, la, lb = (w.reshape(B, -1).contiguous() for w in weights)
    targets = np.array([s.target for s in scheds])
    init_scale, decay = scheds[0].init_scale, scheds[0].decay
    for s in scheds:
        if s.init_scale != init_scale or s.decay != decay:
            raise ValueError("batched problems must share the schedule's init_scale and decay")

    def factor(t):
        return max(1.0, init_scale * decay ** t)

    def eps_vec(t):
        return targets * factor(t)

    f = torch.zeros((B, n), dtype=torch.float32, device=dev)
    fn = torch.zeros_like(f)
    g = torch.zeros((B, m), dtype=torch.float32, device=dev)
    if g_init is not None:
        g.copy_(as_device_f32(g_init).reshape(B, m))
    f_fin = torch.zeros_like(f)
    g_fin = torch.zeros_like(g)
    bias_x = torch.empty_like(f)
    bias_y = torch.empty_like(g)
    first_bad = torch.full((B,), 2 ** 31 - 1, dtype=torch.int32, device=dev)
    active = torch.ones(B, dtype=torch.int32, device=dev)
    host_active = np.ones(B, dtype=bool)
    chk = torch.zeros((B, 8), dtype=torch.float64, device=dev)
    max_checks = max_iters // inner_iters + 2
    err_tab = np.zeros((B, max_checks))
    dual_tab = np.zeros((B, max_checks))
    n_rec = np.zeros(B, dtype=int)
    iters = np.zeros(B, dtype=int)
    conv = np.zeros(B, dtype=bool)

    def dev_f32(v):
        return torch.tensor(np.asarray(v, dtype=np.float32), device=dev)

    e0 = eps_vec(0)
    eps_d = dev_f32(e0)
    kap_d = dev_f32(_LOG2E / e0)
    # initial bias of the column side: g * kappa (per problem); zero for a cold start
    if g_init is None:
        bias_y.zero_()
    else:
        for bb in range(B):
            N.check(lib.otk_make_bias(N.ptr(g[bb]), m, float(np.float32(_LOG2E / e0[bb])),
                                      N.ptr(bias_y[bb]), N.ptr(first_bad[bb:bb + 1]), 1, st))
    f_ready = False
    cur_fac = factor(0)

    def rows(out, kap_next_d, step):
        N.check(lib.otk_dense_lse(N.ptr(C), B, n, m, 0, N.ptr(bias_y), N.ptr(la), N.OTK_FIN_SOLVER,
                                  N.ptr(eps_d), N.ptr(kap_next_d), N.ptr(active), N.ptr(out),
                                  N.ptr(bias_x), N.ptr(first_bad), step, st), "dense rows")

    def cols(kap_next_d, step):
        N.check(lib.otk_dense_lse(N.ptr(CT), B, m, n, 0, N.ptr(bias_x), N.ptr(lb), N.OTK_FIN_SOLVER,
                                  N.ptr(eps_d), N.ptr(kap_next_d), N.ptr(active), N.ptr(g),
                                  N.ptr(bias_y), N.ptr(first_bad), step, st), "dense cols")

    def freeze(idx_np):
        idx = torch.as_tensor(idx_np.astype(np.int64), device=dev)
        f_fin.index_copy_(0, idx, f.index_select(0, idx))
        g_fin.index_copy_(0, idx, g.index_select(0, idx))

    t = 0
    for t in range(1, max_iters + 1):
        fac = factor(t - 1)
        if fac != cur_fac:
            cur_fac = fac
            e = eps_vec(t - 1)
            eps_d = dev_f32(e)
            kap_d = dev_f32(_LOG2E / e)
        fac_next = factor(t)
        kap_next_d = kap_d if fac_next == fac else dev_f32(_LOG2E / eps_vec(t))
        if not f_ready:
            rows(f, kap_d, 2 * t)
        f_ready = False
        cols(kap_next_d, 2 * t + 1)
        if t % inner_iters == 0 or t == max_iters:
            measure = not (fac > 1.0)
            if measure:
                rows(fn, kap_d, 2 * t + 2)
            N.check(lib.otk_check_batched(N.ptr(f), N.ptr(fn) if measure else None, N.ptr(a), n,
                                          N.ptr(g), N.ptr(b), m, B, N.ptr(eps_d), N.ptr(active),
                                          N.ptr(chk), st), "check")
            out = chk.cpu().numpy()
            fb = first_bad.cpu().numpy()
            act = host_active.copy()
            iters[act] = t
            bad = act & ((fb <= 2 * t) | (measure & (fb == 2 * t + 1)))
            nan = act & ~bad & ((out[:, 4] > 0) | (out[:, 5] > 0))
            if raise_on_fail and bad.any():
                raise ValueError(f"problem {int(np.argmax(bad))}: g contains NaN or +inf entries")
            if raise_on_fail and nan.any():
                raise DivergedError("NaN in Sinkhorn potentials; eps is likely too small "
                                    "for the cost scale", iteration=t)
            done = bad | nan
            if measure:
                rec = act & ~done
                k = n_rec[rec]
                err = out[rec, 0]
                err_tab[rec, k] = err
                dual_tab[rec, k] = out[rec, 2] + out[rec, 3] - eps_vec(t - 1)[rec] * (out[rec, 1] - 1.0)
                n_rec[rec] += 1
                hit = np.zeros(B, dtype=bool)
                hit[rec] = err <= threshold
                conv |= hit
                done |= hit
            if done.any():
                host_active &= ~done
                freeze(np.nonzero(done)[0])
                active.copy_(torch.as_tensor(host_active.astype(np.int32), device=dev))
            if not host_active.any():
                break
            if measure and t < max_iters:
                f, fn = fn, f
                f_ready = True
    rest = np.nonzero(host_active)[0]
    if len(rest):
        iters[rest] = min(t, max_iters)
        freeze(rest)
    fh = f_fin.cpu().numpy().astype(np.float64)
    gh = g_fin.cpu().numpy().astype(np.float64)
    return BatchedSinkhornOutput(fh, gh, err_tab, dual_tab, n_rec, iters, conv, targets, f_fin,
                                 g_fin)


def _dense_persistent(C, weights, eps, threshold, max_iters, inner_iters, g_init=None):
    """B stored-cost problems, one CTA each, the whole loop on the device
    (csrc/dense_solve.cu, otk_solve_dense_batched); same per-problem results,
    iteration counts, traces and failure exceptions as ``_dense_loop``."""
    import torch
    B, n, m = C.shape
    dev = C.device
    a, b, la, lb = (w.reshape(B, -1).contiguous() for w in weights)
    max_checks = max_iters // inner_iters + 2
    eps32 = torch.as_tensor(eps.astype(np.float32), device=dev)
    eps64 = torch.as_tensor(eps.astype(np.float64), device=dev)
    gi = None if g_init is None else as_device_f32(g_init).reshape(B, m).contiguous()
    f_out = torch.empty((B, n), dtype=torch.float32, device=dev)
    g_out = torch.empty((B, m), dtype=torch.float32, device=dev)
    errs = torch.zeros((B, max_checks), dtype=torch.float64, device=dev)
    duals = torch.zeros_like(errs)
    state = torch.zeros((B, 5), dtype=torch.int32, device=dev)
    grid = int(os.environ.get("OTK_DENSE_GRID", "0"))
    N.check(N.lib().otk_solve_dense_batched(
        N.ptr(C), B, n, m, N.ptr(a), N.ptr(b), N.ptr(la), N.ptr(lb), N.ptr(eps32), N.ptr(eps64),
        N.ptr(gi), float(threshold), int(max_iters), int(inner_iters), max_checks, N.ptr(f_out),
        N.ptr(g_out), N.ptr(errs), N.ptr(duals), N.ptr(state), grid, stream()),
        "solve_sinkhorn_batched")
    st = state.cpu().numpy()
    failed = np.nonzero(st[:, 3] != N.OTK_OK)[0]
    if len(failed):
        k = failed[np.argmin(st[failed, 4])]
        if st[k, 3] == N.OTK_BAD_POTENTIAL:
            raise ValueError(f"problem {k}: g contains NaN or +inf entries")
        raise DivergedError("NaN in Sinkhorn potentials; eps is likely too small for the cost scale",
                            iteration=int(st[k, 4]))
    return BatchedSinkhornOutput(f_out, g_out, errs, duals, st[:, 0].copy(), st[:, 1].copy(),
                                 st[:, 2].astype(bool), np.asarray(eps, dtype=float), f_out, g_out)


_UNIFORM_CACHE: dict = {}


class _LazyUniform:
    """Host view of uniform batched weights, built only if a caller needs it."""

    def __init__(self, B, size):
        self.B, self.size = B, size

    def __getitem__(self, k):
        return np.full(self.size, 1.0 / self.size)


def solve_sinkhorn_batched(x, y, eps, a=None, b=None, *, threshold: float = 1e-3,
                           max_iters: int = 2000, inner_iters: int = 10, return_cost: bool = False,
                           g_init=None, fixed_iters: bool = False):
    """Solve B independent point-cloud problems with a materialised cost (cfg3).

    x: [B,n,d], y: [B,m,d] (numpy or CUDA tensors); eps: scalar or [B];
    a: [B,n] / b: [B,m] or None (uniform); g_init: [B,m] warm start (the
    reference's inner-solve use, quadratic.py:169-177).  Builds C[B,n,m] on the GPU
    (otk_dense_cost), then runs the lock-step dense loop.  Returns a list of
    SinkhornOutput (and the RegOTCost list when ``return_cost``).
    """
    import torch
    device()
    if max_iters < 1 or inner_iters < 1:
        raise ValueError("max_iters and inner_iters must be >= 1")
    if not (threshold > 0):
        raise ValueError("threshold must be positive")
    if fixed_iters:  # measurement knob, as in solve_sinkhorn: the checks never stop the loop
        threshold = -1.0
    xd = as_device_f32(x)
    yd = as_device_f32(y)
    if xd.ndim != 3 or yd.ndim != 3 or xd.shape[0] != yd.shape[0] or xd.shape[2] != yd.shape[2]:
        raise ValueError("x and y must be [B,n,d] and [B,m,d]")
    B, n, d = xd.shape
    m = yd.shape[1]
    eps = np.broadcast_to(np.asarray(eps, dtype=float), (B,))
    if not np.all(eps > 0):
        raise ValueError("eps must be positive")
    _fp32_guard(EpsilonSchedule(float(eps.min())), inner_iters, max_iters)
    dev = xd.device

    def weights_of(w, size, name):
        if w is None:  # uniform: built on the device once per shape (read-only)
            key = (B, size, str(dev))
            if key not in _UNIFORM_CACHE:
                u = torch.full((B, size), 1.0 / size, dtype=torch.float32, device=dev)
                _UNIFORM_CACHE.clear()
                _UNIFORM_CACHE[key] = (u, torch.full_like(u, float(-np.log(size))))
            u, lu = _UNIFORM_CACHE[key]
            return _LazyUniform(B, size), u, lu
        ww = np.stack([_as_weights(w[k], size, name) for k in range(B)])
        with np.errstate(divide="ignore"):
            return ww, as_device_f32(ww), as_device_f32(np.log(ww))
    aw, a_d, la_d = weights_of(a, n, "a")
    bw, b_d, lb_d = weights_of(b, m, "b")
    persistent = bool(N.lib().otk_dense_solve_fits(n, m)) and not os.environ.get("OTK_DENSE_LOCKSTEP")
    C = torch.empty((B, n, m), dtype=torch.float32, device=dev)
    CT = None if persistent else torch.empty((B, m, n), dtype=torch.float32, device=dev)
    N.check(N.lib().otk_dense_cost(N.ptr(xd), N.ptr(yd), B, n, m, d, 0, N.ptr(C), N.ptr(CT),
                                   stream()), "dense_cost")
    with nvtx_range("otk batched solve"):
        if persistent:
            outs = _dense_persistent(C, (a_d, b_d, la_d, lb_d), np.asarray(eps, dtype=float), threshold,
                                     max_iters, inner_iters, g_init)
        else:
            scheds = [EpsilonSchedule(float(e)) for e in eps]
            outs = _dense_loop(C, CT, (a_d, b_d, la_d, lb_d), scheds, threshold, max_iters,
                               inner_iters, g_init=g_init)
    if not return_cost:
        return outs
    costs = _dense_costs(C, outs, aw, bw)
    return outs, costs


def _dense_costs(C, outs, aw, bw):
    import torch
    B, n, m = C.shape
    f, g = outs.f_device, outs.g_device
    eps = torch.as_tensor(np.asarray(outs.eps, dtype=np.float32), device=C.device)
    res = torch.zeros((B, 2), dtype=torch.float64, device=C.device)
    N.check(N.lib().otk_dense_cost_reduce(N.ptr(C), B, n, m, N.ptr(f), N.ptr(g), N.ptr(eps),
                                          N.ptr(res), stream()), "dense_cost_reduce")
    r = res.cpu().numpy()
    return [RegOTCost(float(r[k, 0]), _dual_objective(outs.f[k], outs.g[k], aw[k], bw[k],
                                                      float(outs.eps[k]), float(r[k, 1])))
            for k in range(B)]


# ---------------------------------------------------------------- post-solve
def transport_matrix(out: SinkhornOutput, prob: LinearProblem) -> Coupling:
    """exp((f + g - C)/eps) materialised on the GPU (sinkhorn.py:203-207); keeps the cap."""
    import torch
    geom = prob.geom
    geom._check_cap(None)
    n, m = geom.shape
    f = as_device_f32(out.f_device if out.f_device is not None else out.f)
    g = as_device_f32(out.g_device if out.g_device is not None else out.g)
    if isinstance(geom, PointCloudGeometry):
        cx, cy = geom._clouds()
        plan = torch.empty((n, m), dtype=torch.float32, device=cx.p.device)
        N.check(N.lib().otk_transport_matrix(N.ptr(cx.p), N.ptr(cx.sq), n, N.ptr(cy.p), N.ptr(cy.sq),
                                             m, cx.d, N.ptr(f), N.ptr(g), float(out.eps),
                                             geom._cost_flags, N.ptr(plan), stream()),
                "transport_matrix")
    elif isinstance(geom, DenseGeometry):
        C = geom._c()
        plan = torch.empty((n, m), dtype=torch.float32, device=C.device)
        N.check(N.lib().otk_dense_plan(N.ptr(C), n, m, N.ptr(f), N.ptr(g), float(out.eps),
                                       N.ptr(plan), stream()), "transport_matrix")
    else:
        raise TypeError(f"unsupported geometry {type(geom).__name__}")
    return Coupling(plan.cpu().numpy().astype(np.float64))


def reg_ot_cost(out: SinkhornOutput, prob: LinearProblem) -> RegOTCost:
    """<C, P> and the dual objective (sinkhorn.py:210-216), computed online on the GPU."""
    import torch
    geom = prob.geom
    n, m = geom.shape
    f = as_device_f32(out.f_device if out.f_device is not None else out.f)
    g = as_device_f32(out.g_device if out.g_device is not None else out.g)
    if isinstance(geom, PointCloudGeometry):
        cx, cy = geom._clouds()
        lib = N.lib()
        ws = torch.empty(lib.otk_cost_workspace_bytes(n, m), dtype=torch.uint8, device=cx.p.device)
        res = torch.zeros(2, dtype=torch.float64, device=cx.p.device)
        N.check(lib.otk_cost_partial(N.ptr(cx.p), N.ptr(cx.sq), n, N.ptr(cy.p), N.ptr(cy.sq), m,
                                     cx.d, N.ptr(f), N.ptr(g), float(out.eps), geom._cost_flags,
                                     N.ptr(res), N.ptr(ws), stream()), "reg_ot_cost")
        transport, mass = (float(v) for v in res.cpu().numpy())
    elif isinstance(geom, DenseGeometry):
        C = geom._c()
        res = torch.zeros(2, dtype=torch.float64, device=C.device)
        eps_t = torch.tensor([out.eps], dtype=torch.float32, device=C.device)
        N.check(N.lib().otk_dense_cost_reduce(N.ptr(C), 1, n, m, N.ptr(f), N.ptr(g), N.ptr(eps_t),
                                              N.ptr(res), stream()), "reg_ot_cost")
        transport, mass = (float(v) for v in res.cpu().numpy())
    else:
        raise TypeError(f"unsupported geometry {type(geom).__name__}")
    fh = out.f if not is_torch(out.f) else out.f.double().cpu().numpy()
    gh = out.g if not is_torch(out.g) else out.g.double().cpu().numpy()
    return RegOTCost(transport, _dual_objective(fh, gh, prob.a, prob.b, out.eps, mass))


def grad_weights(out: SinkhornOutput, prob: LinearProblem) -> np.ndarray:
    """Envelope gradient in a: centred f (sinkhorn.py:219-229)."""
    if not out.converged:
        raise ValueError("grad_weights requires a converged solution")
    return out.f - out.f.mean()


def grad_points(out: SinkhornOutput, prob: LinearProblem):
    """Envelope gradient in x: 2(rowmass*x - P y) (sinkhorn.py:232-246).

    Computed online on the GPU (otk_grad_points): the plan is rebuilt tile by
    tile and never stored, so unlike the reference (which materialises it
    through transport_matrix) there is no n*m cap.  numpy in -> float64 numpy
    out; CUDA tensors in -> float32 CUDA tensor out.
    """
    import torch
    if not out.converged:
        raise ValueError("grad_points requires a converged solution")
    geom = prob.geom
    if not isinstance(geom, PointCloudGeometry) or geom.cost_fn != "sqeucl":
        raise ValueError("grad_points requires a PointCloudGeometry with the sqeucl cost")
    cx, cy = geom._clouds()
    n, m = geom.shape
    f = as_device_f32(out.f_device if out.f_device is not None else out.f)
    g = as_device_f32(out.g_device if out.g_device is not None else out.g)
    grad = torch.empty((n, cx.d), dtype=torch.float32, device=cx.p.device)
    N.check(N.lib().otk_grad_points(N.ptr(cx.p), N.ptr(cx.sq), n, N.ptr(cy.p), N.ptr(cy.sq), m,
                                    cx.d, N.ptr(f), N.ptr(g), float(out.eps),
                                    N.OTK_SAME_POINTS if geom._same_points else 0, N.ptr(grad),
                                    stream()), "grad_points")
    return to_output(grad, geom.x)
