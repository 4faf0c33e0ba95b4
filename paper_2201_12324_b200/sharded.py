"""Row-sharded multi-GPU Sinkhorn (no reference equivalent).

The reference loop (sinkhorn.py:151-200) is single-process.  Here x (with f
and the weights a) is split into W contiguous row shards, one per rank /
GPU; y, g and b are replicated:

* f half-step (sinkhorn.py:173) reduces over j -- all of g is local, so it is
  a plain local ``otk_lse_partial`` + ``otk_lse_finalize``.
* g half-step (sinkhorn.py:174) reduces over i -- each rank reduces its own
  rows into one log2-partial per column (``otk_lse_partial`` +
  ``otk_lse_finalize(mode=OTK_FIN_LOG2)``), the W partials are all-gathered
  (NCCL over NVLink; m floats per rank) and every rank combines them in rank
  order with the same finalize kernel, so g stays bitwise identical on all
  ranks and a 1-rank run is bitwise identical to the single-GPU solver.
* the check (sinkhorn.py:175-189) runs the fused check kernel on the local
  rows; the 8 partial sums are all-gathered and added in rank order on the
  host, so every rank takes the same converged / diverged decision.

The loop itself (``sharded_loop``) is host logic over two small interfaces:
an *engine* (the device half-steps: ``CudaShardEngine``, the sm_100a library)
and a *comm* (``TorchComm`` = ``torch.distributed``; ``ThreadComm`` = ranks
emulated by threads of one process, for single-GPU tests).  The CPU tests
drive the same loop with a float64 numpy engine over ``gloo``.
"""

from __future__ import annotations

import dataclasses
import os
import threading

import numpy as np

from . import _native as N
from ._device import as_device_f32, device, nvtx_range, stream
from .errors import DivergedError
from .geometry import EpsilonSchedule

__all__ = [
    "shard_rows",
    "ShardedSinkhornOutput",
    "TorchComm",
    "ThreadComm",
    "CudaShardEngine",
    "sharded_loop",
    "ShardedProblem",
    "PeerExchange",
    "solve_sinkhorn_sharded",
    "reg_ot_cost_sharded",
]

_LOG2E = 1.4426950408889634


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row range [lo, hi) of ``rank`` (first n % world shards get +1)."""
    if not (0 <= rank < world):
        raise ValueError("rank must lie in [0, world)")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclasses.dataclass(frozen=True, eq=False)
class ShardedSinkhornOutput:
    f_local: np.ndarray          # this rank's rows of f (float64)
    g: np.ndarray                # replicated (float64)
    errors: np.ndarray
    dual_trace: np.ndarray
    iterations: int
    converged: bool
    eps: float
    row_offset: int
    n_total: int
    f: np.ndarray | None = None  # all rows (gather_f=True)
    f_device: object = dataclasses.field(default=None, repr=False)
    g_device: object = dataclasses.field(default=None, repr=False)


# ---------------------------------------------------------------- comms
class TorchComm:
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_rows(self, local):
        import torch
        shape_dev = local.device
        local = local.contiguous().reshape(-1)
        if local.is_cuda and self.dist.get_backend(self.group) == "gloo":
            local = local.cpu()  # gloo moves host tensors
        out = torch.empty(self.world * local.numel(), dtype=local.dtype, device=local.device)
        self.dist.all_gather_into_tensor(out, local, group=self.group)
        return out.view(self.world, -1).to(shape_dev)

    def _host(self, arr, like_device):
        import torch
        return torch.as_tensor(np.asarray(arr, dtype=np.float64), device=like_device)

    def all_gather_host(self, vec: np.ndarray, device) -> np.ndarray:
        """[k] float64 per rank -> [world, k] on every rank (collective on ``device``)."""
        t = self._host(vec, device)
        return self.all_gather_rows(t).cpu().numpy()

    def all_gather_objects(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def all_gather_bytes(self, b: bytes) -> list:
        return [bytes(x) for x in self.all_gather_objects(bytes(b))]


class ThreadComm:
    """W ranks emulated by W threads of one process (shared device, host barrier).

    Used to run the sharded loop on one GPU: no kernel ever waits on another
    rank's kernel -- every exchange goes through the host after a stream sync.
    """

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.shared = shared
        self.rank = rank
        self.world = shared.world

    @classmethod
    def group(cls, world: int):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _exchange(self, obj):
        sh = self.shared
        sh.barrier.wait()
        sh.slots[self.rank] = obj
        sh.barrier.wait()
        out = list(sh.slots)
        sh.barrier.wait()
        return out

    def all_gather_rows(self, local):
        import torch
        if local.is_cuda:
            torch.cuda.current_stream(local.device).synchronize()
        parts = self._exchange(local)
        out = torch.stack([p.to(local.device) for p in parts])
        if local.is_cuda:  # every copy done before any rank overwrites its buffer
            torch.cuda.current_stream(local.device).synchronize()
        self.shared.barrier.wait()
        return out

    def all_gather_host(self, vec: np.ndarray, device=None) -> np.ndarray:
        return np.stack(self._exchange(np.asarray(vec, dtype=np.float64).copy()))


# ---------------------------------------------------------------- peer-memory exchange
class PeerExchange:
    """The g half-step's exchange over NVLink peer memory (csrc/p2p.cu).

    Every rank allocates one exchange buffer, exports it as a CUDA IPC handle,
    opens the other ranks' handles (handles travel through ``comm``'s host
    all-gather) and writes the W base pointers into its own buffer.  Each g
    half-step then pushes its column partials from the half-step's last
    kernel and combines the W partials after per-block acquire flags (see
    include/otk.h, otk_exchange).  One process per GPU only: ranks that share
    a GPU (``ThreadComm``) must not run kernels that wait on each other.
    """

    _CACHE: dict = {}

    @classmethod
    def shared(cls, comm, m: int) -> "PeerExchange":
        """One exchange buffer per (process group, m): built (IPC handles
        exported, opened and exchanged) on first use, reused by every later
        ShardedProblem on the same group -- the epoch sequence continues."""
        key = (id(getattr(comm, "group", None)), comm.world, comm.rank, int(m))
        px = cls._CACHE.get(key)
        if px is None or px.local is None:
            px = cls._CACHE[key] = cls(comm, m)
        return px

    def __init__(self, comm, m: int):
        import ctypes
        lib = N.lib()
        self.world, self.rank, self.m = comm.world, comm.rank, int(m)
        self.bytes = lib.otk_exchange_bytes(self.world, self.m)
        buf = ctypes.c_void_p()
        N.check(lib.otk_exchange_alloc(self.bytes, ctypes.byref(buf)), "exchange alloc")
        self.local = buf.value
        self.opened = []
        try:
            handle = (ctypes.c_uint8 * 64)()
            N.check(lib.otk_ipc_handle(self.local, handle), "ipc handle")
            handles = comm.all_gather_bytes(bytes(handle))
            ptrs = []
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self.local)
                    continue
                peer = ctypes.c_void_p()
                N.check(lib.otk_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(h),
                                         ctypes.byref(peer)), f"ipc open (rank {r})")
                self.opened.append(peer.value)
                ptrs.append(peer.value)
            table = (ctypes.c_void_p * self.world)(*ptrs)
            N.check(lib.otk_exchange_set_peers(self.local, self.world, self.m, table, stream()),
                    "exchange peers")
        except Exception:
            self.close()
            raise
        self.epoch = 0

    def next(self):
        """Arguments of the next exchange.  Epoch 0 = device-counted: the buffer
        itself numbers the exchanges (the combine kernel advances the count), so
        the Python loop and the native solver (and its CUDA graphs) share one
        epoch sequence; ``epoch`` here only counts this object's exchanges."""
        self.epoch += 1
        return N.Exchange(self.local, self.world, self.rank, 0)

    def args(self):
        """otk_exchange for the native sharded solver (device-counted epochs)."""
        return N.Exchange(self.local, self.world, self.rank, 0)

    def status(self) -> int:
        import ctypes
        v = ctypes.c_int32()
        N.check(N.lib().otk_exchange_status(self.local, ctypes.byref(v), stream()), "exchange status")
        return int(v.value)

    def close(self):
        lib = N.lib()
        for p in self.opened:
            lib.otk_ipc_close(p)
        self.opened = []
        if getattr(self, "local", None):
            lib.otk_exchange_free(self.local)
            self.local = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def p2p_exchange_supported(comm) -> bool:
    """True when every rank is a separate process on its own GPU of one host and
    every pair of those GPUs can access each other's memory (NVLink / NVSwitch)."""
    import socket
    import torch
    if not isinstance(comm, TorchComm) or comm.dist.get_backend(comm.group) != "nccl":
        return False
    me = (socket.gethostname(), torch.cuda.current_device())
    everyone = comm.all_gather_objects(me)
    if len({h for h, _ in everyone}) != 1 or len({d for _, d in everyone}) != len(everyone):
        return False
    dev = me[1]
    return all(d == dev or torch.cuda.can_device_access_peer(dev, d) for _, d in everyone)


# ---------------------------------------------------------------- device engine
class CudaShardEngine:
    """Device half-steps of one rank (libotk_sm100.so), mirroring solve.cu's HalfStep."""

    def __init__(self, x_local, y, a_local, b, flags: int = 0, amax_reduce=None):
        """``amax_reduce(local_amax) -> global_amax`` makes the split-fp16 operand
        scale common to all ranks (None: this rank's own)."""
        import torch
        from .geometry import _Cloud
        device()
        self.cx = _Cloud(x_local)
        self.cy = _Cloud(y)
        if self.cx.d != self.cy.d:
            raise ValueError("x and y must have the same dimension")
        self.n, self.m, self.d = self.cx.n, self.cy.n, self.cx.d
        lib = N.lib()
        planes = bool(lib.otk_lse_uses_tc(self.d, flags))
        scale = 1.0
        if planes:
            amax = max(self.cx.absmax(), self.cy.absmax())
            if amax_reduce is not None:
                amax = amax_reduce(amax)
            scale = float(lib.otk_split_scale(amax, self.d))
        self.cx.prepare(scale, planes)
        self.cy.prepare(scale, planes)
        self.sinv = 1.0 / (scale * scale)
        self.flags = (flags & (N.OTK_IMPL_SIMT | N.OTK_IMPL_TC | N.OTK_COST_EUCL)) | N.OTK_CLAMP
        dev = self.cx.p.device
        with np.errstate(divide="ignore"):
            la, lb = np.log(np.asarray(a_local, dtype=np.float64)), np.log(np.asarray(b, dtype=np.float64))
        self.a, self.b = as_device_f32(a_local), as_device_f32(b)
        self.la, self.lb = as_device_f32(la), as_device_f32(lb)
        self.nsr = lib.otk_lse_suggest_nsplit(self.n, self.m, self.d, self.flags)
        self.nsc = lib.otk_lse_suggest_nsplit(self.m, self.n, self.d, self.flags)
        f32 = dict(dtype=torch.float32, device=dev)
        self.part = torch.empty(max(self.nsr * self.n, self.nsc * self.m), **f32)
        self.f = [torch.zeros(self.n, **f32), torch.zeros(self.n, **f32)]
        self.g = torch.zeros(self.m, **f32)
        self.bias_x = torch.empty(self.n, **f32)
        self.bias_y = torch.empty(self.m, **f32)
        self.lcol = torch.empty(self.m, **f32)
        self.first_bad = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=dev)
        self.chk = torch.zeros(8, dtype=torch.float64, device=dev)
        self.chk_ws = torch.zeros(lib.otk_check_workspace_bytes(), dtype=torch.uint8, device=dev)
        self.device = dev
        self.launches = 0
        # anchored half-steps (otk_lse_step): per-role anchors + repair workspaces
        self.anchored = bool(lib.otk_lse_step_anchored(self.n, self.m, self.d, self.flags)) and not (
            flags & N.OTK_IMPL_NOANCHOR)
        self.anc_x = torch.empty(self.n, **f32)
        self.anc_y = torch.empty(self.m, **f32)
        self.rep_x = torch.empty(lib.otk_lse_step_workspace_bytes(self.n), dtype=torch.uint8, device=dev)
        self.rep_y = torch.empty(lib.otk_lse_step_workspace_bytes(self.m), dtype=torch.uint8, device=dev)
        self.have_x = self.have_y = False

    def set_g(self, g_init, kappa):
        if g_init is None:
            self.g.zero_()
        else:
            self.g.copy_(as_device_f32(g_init))
        N.check(N.lib().otk_make_bias(N.ptr(self.g), self.m, kappa, N.ptr(self.bias_y),
                                      N.ptr(self.first_bad), 1, stream()), "make_bias")

    def _launches(self, have):
        return 4 if (self.anchored and have) else 2

    def rows(self, kappa, eps, kappa_next, which, step):
        """Local f half-step (otk_lse_step: partial + finalize, anchored after the first)."""
        cx, cy, lib = self.cx, self.cy, N.lib()
        fl = self.flags | (0 if self.have_x else N.OTK_ANCHOR_INIT)
        N.check(lib.otk_lse_step(N.ptr(cx.p), N.ptr(cx.sq), N.ptr(cx.hi), N.ptr(cx.lo),
                                 N.ptr(cx.ext_a), self.n, N.ptr(cy.p), N.ptr(cy.sq), N.ptr(cy.hi),
                                 N.ptr(cy.lo), N.ptr(cy.ext_b), self.m, self.d, cx.dpad,
                                 self.sinv, N.ptr(self.bias_y), kappa, fl, self.nsr,
                                 N.ptr(self.part), N.ptr(self.la), N.OTK_FIN_SOLVER, eps, kappa_next,
                                 N.ptr(self.f[which]), N.ptr(self.bias_x), N.ptr(self.first_bad), step,
                                 N.ptr(self.anc_x) if self.anchored else None, N.ptr(self.rep_x),
                                 None, stream()), "rows half-step")
        self.launches += self._launches(self.have_x)
        self.have_x = True

    def cols_partial(self, kappa, xchg=None):
        """This shard's log2 column partials (OTK_FIN_LOG2), anchored on the shard's own
        previous partials; with ``xchg`` (an ``N.Exchange``) the last finalize kernel
        also pushes them into every rank's exchange buffer over peer memory."""
        import ctypes
        cx, cy, lib = self.cx, self.cy, N.lib()
        fl = self.flags | (0 if self.have_y else N.OTK_ANCHOR_INIT)
        N.check(lib.otk_lse_step(N.ptr(cy.p), N.ptr(cy.sq), N.ptr(cy.hi), N.ptr(cy.lo),
                                 N.ptr(cy.ext_a), self.m, N.ptr(cx.p), N.ptr(cx.sq), N.ptr(cx.hi),
                                 N.ptr(cx.lo), N.ptr(cx.ext_b), self.n, self.d, cx.dpad,
                                 self.sinv, N.ptr(self.bias_x), kappa, fl, self.nsc,
                                 N.ptr(self.part), None, N.OTK_FIN_LOG2, 0.0, 0.0,
                                 N.ptr(self.lcol), None, None, 0,
                                 N.ptr(self.anc_y) if self.anchored else None, N.ptr(self.rep_y),
                                 ctypes.byref(xchg) if xchg is not None else None, stream()),
                "cols half-step")
        self.launches += self._launches(self.have_y)
        self.have_y = True
        return self.lcol

    def cols_exchange(self, p2p, kappa, eps, kappa_next, step):
        """g half-step over peer memory: local partials pushed to every rank by the
        half-step's last kernel, then the W partials combined in rank order."""
        x = p2p.next()
        self.cols_partial(kappa, x)
        N.check(N.lib().otk_exchange_finalize(x.local, x.world, self.m, x.epoch, N.ptr(self.lb),
                                              N.OTK_FIN_SOLVER, eps, kappa_next, N.ptr(self.g),
                                              N.ptr(self.bias_y), N.ptr(self.first_bad), step, 0,
                                              stream()), "exchange combine")
        self.launches += 1

    def cols_finalize(self, lall, eps, kappa_next, step):
        W = lall.shape[0]
        N.check(N.lib().otk_lse_finalize(N.ptr(lall), W, self.m, N.ptr(self.lb), N.OTK_FIN_SOLVER,
                                         eps, kappa_next, N.ptr(self.g), N.ptr(self.bias_y),
                                         N.ptr(self.first_bad), step, stream()), "combine")
        self.launches += 1

    def check(self, which, measure, eps):
        fn = self.f[1 - which] if measure else None
        N.check(N.lib().otk_check(N.ptr(self.f[which]), N.ptr(fn), N.ptr(self.a), self.n,
                                  N.ptr(self.g), N.ptr(self.b), self.m, eps, N.ptr(self.chk),
                                  N.ptr(self.chk_ws), stream()), "check")
        self.launches += 1
        return self.chk.cpu().numpy().copy()

    def read_first_bad(self) -> int:
        return int(self.first_bad.item())

    def reset_first_bad(self):
        self.first_bad.fill_(2 ** 31 - 1)

    def f_result(self, which):
        return self.f[which]

    def g_result(self):
        return self.g


# ---------------------------------------------------------------- the loop
def sharded_loop(engine, comm, sched: EpsilonSchedule, threshold: float, max_iters: int,
                 inner_iters: int, g_init=None, p2p=None):
    """The reference loop (sinkhorn.py:151-200) over row shards.

    The g half-step's exchange goes through ``comm`` (all-gather of the column
    partials, e.g. NCCL) or, with ``p2p`` (a ``PeerExchange``), over peer
    memory from the half-step's own last kernel.

    Returns (which_f, iterations, converged, errors, duals).  Raises
    DivergedError / ValueError at the same iteration the single-GPU solver
    (solve.cu) would.  Same step numbering as solve.cu: the finalize of f_t
    records step 2t, g_t records 2t+1, the check's f_{t+1} records 2t+2.
    """
    target = sched.target
    engine.set_g(g_init, float(np.float32(_LOG2E / sched.at(0))))
    which, f_ready = 0, False
    errors, duals = [], []
    converged = False
    t = 0
    for t in range(1, max_iters + 1):
        e = sched.at(t - 1)
        kap = float(np.float32(_LOG2E / e))
        kap_next = float(np.float32(_LOG2E / sched.at(t)))
        if not f_ready:
            with nvtx_range("otk sharded f half-step"):
                engine.rows(kap, e, kap, which, 2 * t)
        f_ready = False
        with nvtx_range("otk sharded g half-step + exchange"):
            if p2p is not None:  # fused push (last kernel of the half-step) + combine
                engine.cols_exchange(p2p, kap, e, kap_next, 2 * t + 1)
            else:
                lall = comm.all_gather_rows(engine.cols_partial(kap))
                engine.cols_finalize(lall, e, kap_next, 2 * t + 1)
        if t % inner_iters == 0 or t == max_iters:
            measure = not (e > target)
            with nvtx_range("otk sharded check"):
                if measure:
                    engine.rows(kap, e, kap, 1 - which, 2 * t + 2)
                local = engine.check(which, measure, e)
            fb = engine.read_first_bad()
            # this rank's exchange status travels with its sums: a timed-out peer
            # wait makes EVERY rank raise at the same check (none is left waiting
            # in the gather below)
            xs = float(p2p.status()) if p2p is not None else 0.0
            rows = comm.all_gather_host(np.concatenate([local, [float(fb), xs]]), engine.device)
            if rows[:, 9].max() != 0.0:
                raise RuntimeError("peer-memory exchange timed out waiting for another rank")
            tot = np.zeros(8)
            for r in range(rows.shape[0]):          # fixed rank order: deterministic
                tot += rows[r, :8]
            for k in (3, 5, 7):                      # g terms are replicated: count once
                tot[k] = rows[0, k]
            fb = int(rows[:, 8].min())
            if fb <= 2 * t:
                raise ValueError(f"g contains NaN or +inf entries (potential fed to iteration "
                                 f"{(fb + 1) // 2})")
            if tot[4] > 0 or tot[5] > 0:
                raise DivergedError("NaN in Sinkhorn potentials; eps is likely too small for the "
                                    "cost scale", iteration=t)
            if not measure:
                continue
            if fb == 2 * t + 1:
                raise ValueError(f"g contains NaN or +inf entries (potential fed to iteration {t})")
            err = float(tot[0])
            errors.append(err)
            duals.append(float(tot[2] + tot[3] - e * (tot[1] - 1.0)))
            if err <= threshold:
                converged = True
                break
            if t < max_iters:
                which, f_ready = 1 - which, True
    if p2p is not None and p2p.status() != 0:
        raise RuntimeError("peer-memory exchange timed out waiting for another rank")
    return which, min(t, max_iters), converged, np.asarray(errors), np.asarray(duals)


def _global_weights(w, n_total, lo, hi, name):
    if w is None:
        return np.full(hi - lo, 1.0 / n_total)
    w = np.asarray(w.detach().double().cpu().numpy() if hasattr(w, "detach") else w, dtype=float)
    if w.shape == (n_total,):
        w = w[lo:hi]
    if w.shape != (hi - lo,):
        raise ValueError(f"{name} must have shape ({n_total},) or the shard's ({hi - lo},)")
    if not np.all(np.isfinite(w)) or np.any(w < 0):
        raise ValueError(f"{name} must be entrywise finite and nonnegative")
    return w


class ShardedProblem:
    """One rank's share of a row-sharded point-cloud problem, prepared once.

    ``x``: the full [n, d] points (each rank takes its ``shard_rows`` slice) or,
    with ``x_is_local``, this rank's rows (then pass ``n_total``).  ``y`` [m, d],
    ``b`` [m] replicated; ``a`` global [n] (or the local slice).  ``comm``:
    ``TorchComm()`` (default; needs an initialised process group) or a
    ``ThreadComm``.  Construction validates the weights, uploads and prepares
    the points (norms, split-fp16 planes with one scale common to all ranks);
    ``solve`` can then be called repeatedly (like reusing a geometry).
    """

    def __init__(self, x, y, a=None, b=None, *, comm=None, x_is_local: bool = False,
                 n_total: int | None = None, impl: str = "auto", cost_fn: str = "sqeucl",
                 exchange: str = "auto"):
        from .geometry import centered_points, cost_fn_flags
        from .sinkhorn import _impl_flags
        cflags = cost_fn_flags(cost_fn)
        self.cost_fn = cost_fn
        self.comm = comm = comm or TorchComm()
        dev = _dev_of(x)
        if x_is_local:
            if n_total is None:
                raise ValueError("n_total is required with x_is_local")
            sizes = comm.all_gather_host(np.array([float(x.shape[0])]), dev)[:, 0].astype(int)
            lo = int(sizes[:comm.rank].sum())
            hi = lo + int(x.shape[0])
            if int(sizes.sum()) != n_total:
                raise ValueError("local shards do not add up to n_total")
            x_local = x
        else:
            n_total = int(x.shape[0])
            lo, hi = shard_rows(n_total, comm.world, comm.rank)
            x_local = x[lo:hi]
        m = int(y.shape[0])
        a_loc = _global_weights(a, n_total, lo, hi, "a")
        b_w = _global_weights(b, m, 0, m, "b")
        tot_a = comm.all_gather_host(np.array([a_loc.sum()]), dev)[:, 0].sum()
        if abs(tot_a - 1.0) > 1e-8 or abs(b_w.sum() - 1.0) > 1e-8:
            raise ValueError("a and b must each sum to 1")

        def amax_reduce(v):  # one common split scale on every rank
            return float(comm.all_gather_host(np.array([v]), dev)[:, 0].max())

        self._amax_reduce = amax_reduce
        kx, ky = centered_points(x_local, y, cost_fn)  # common centre: the replicated y's median
        self.kx, self.ky = kx, ky
        self.a_loc, self.b_w = a_loc, b_w
        self.flags = _impl_flags(impl) | cflags
        self._engine = None
        self._native = None
        self.lo, self.hi, self.n_total, self.m = lo, hi, n_total, m
        # g half-step exchange: "p2p" = pushed over NVLink peer memory by the
        # half-step's last kernel (csrc/p2p.cu); "collective" = comm all-gather
        # (NCCL) + combine; "auto" = p2p whenever every rank is its own process
        # on its own peer-accessible GPU of one host (OTK_EXCHANGE overrides)
        exchange = os.environ.get("OTK_EXCHANGE", exchange)
        if exchange not in ("auto", "p2p", "collective"):
            raise ValueError("exchange must be 'auto', 'p2p' or 'collective'")
        self.p2p = None
        if exchange != "collective":
            ok = p2p_exchange_supported(comm)
            if exchange == "p2p" and not ok:
                raise ValueError("peer-memory exchange needs one process per GPU of one host "
                                 "(TorchComm over NCCL) with peer access between all GPUs")
            if ok:
                self.p2p = PeerExchange.shared(comm, m)
        self.exchange = "p2p" if self.p2p is not None else "collective"
        # the loop: native C++ (otk_solve_pointcloud_sharded: graph-captured check
        # periods, check sums exchanged on the device, one host sync per check)
        # whenever the exchange is peer memory; the Python loop otherwise
        # (collective / ThreadComm / gloo) or with OTK_SHARDED_LOOP=python
        self.loop = "native" if (self.p2p is not None and
                                 os.environ.get("OTK_SHARDED_LOOP", "native") != "python") else "python"

    @property
    def engine(self) -> "CudaShardEngine":
        """Device half-steps for the Python loop (built on first use)."""
        if self._engine is None:
            self._engine = CudaShardEngine(self.kx, self.ky, self.a_loc, self.b_w, flags=self.flags,
                                           amax_reduce=self._amax_reduce)
        return self._engine

    def _native_state(self):
        """Per-problem state of the native loop, built once: device weights,
        the common operand scale and the solver workspace (reused by every solve)."""
        if self._native is None:
            import torch
            lib = N.lib()
            n, d = self.kx.shape
            m = self.m
            scale = 0.0
            if lib.otk_lse_uses_tc(d, self.flags):
                amax = max(float(_absmax(self.kx)), float(_absmax(self.ky)))
                scale = float(lib.otk_split_scale(self._amax_reduce(amax), d))
            with np.errstate(divide="ignore"):
                la, lb = np.log(self.a_loc), np.log(self.b_w)
            st = dict(a=as_device_f32(self.a_loc), b=as_device_f32(self.b_w), la=as_device_f32(la),
                      lb=as_device_f32(lb), scale=scale, ws=None, ws_key=None)
            n_pad = (n + 63) // 64 * 64
            st["fg"] = torch.empty(n_pad + m, dtype=torch.float32, device=self.kx.device)
            st["n_pad"] = n_pad
            self._native = st
        return self._native

    def _solve_native(self, sched, threshold, max_iters, inner_iters, g_init):
        import ctypes
        import torch
        from .sinkhorn import _raise_status
        st = self._native_state()
        n, d = self.kx.shape
        m = self.m
        max_checks = max_iters // inner_iters + 2
        errs, duals = np.zeros(max_checks), np.zeros(max_checks)
        gi = None
        if g_init is not None:
            gi = as_device_f32(g_init)
            if tuple(gi.shape) != (m,):
                raise ValueError(f"g_init must have shape ({m},)")
        fg, n_pad = st["fg"], st["n_pad"]
        A = N.SolveArgs()
        A.x, A.y, A.n, A.m, A.d = N.ptr(self.kx), N.ptr(self.ky), n, m, d
        A.a, A.b, A.log_a, A.log_b = N.ptr(st["a"]), N.ptr(st["b"]), N.ptr(st["la"]), N.ptr(st["lb"])
        A.same_points = 0
        A.eps_target, A.eps_init_scale, A.eps_decay = sched.target, sched.init_scale, sched.decay
        A.threshold, A.max_iters, A.inner_iters = float(threshold), int(max_iters), int(inner_iters)
        A.g_init = N.ptr(gi)
        A.flags = self.flags | N.OTK_IMPL_NOPERSIST
        A.use_graphs = 1
        A.f_out, A.g_out = N.ptr(fg[:n]), N.ptr(fg[n_pad:])
        A.errors = errs.ctypes.data_as(ctypes.c_void_p)
        A.duals = duals.ctypes.data_as(ctypes.c_void_p)
        A.max_checks = max_checks
        lib = N.lib()
        nbytes = lib.otk_solve_workspace_bytes(ctypes.byref(A))
        if st["ws"] is None or st["ws"].numel() < nbytes:
            st["ws"] = torch.empty(nbytes, dtype=torch.uint8, device=self.kx.device)
        A.workspace, A.workspace_bytes, A.stream = N.ptr(st["ws"]), st["ws"].numel(), stream()
        X = self.p2p.args()
        rc = lib.otk_solve_pointcloud_sharded(ctypes.byref(A), ctypes.byref(X), st["scale"], 0)
        self.launches_last = int(A.launches)
        if rc != N.OTK_OK:
            _raise_status(rc, A.fail_iter)
        k = A.n_checks
        return (fg[:n].clone(), fg[n_pad:].clone(), int(A.iterations), bool(A.converged),
                errs[:k].copy(), duals[:k].copy())

    def solve(self, eps, *, threshold: float = 1e-3, max_iters: int = 2000,
              inner_iters: int = 10, g_init=None, gather_f: bool = False,
              fixed_iters: bool = False) -> ShardedSinkhornOutput:
        """The reference loop (sinkhorn.py:151-200) over the shards; same
        validation and errors as ``solve_sinkhorn`` (``fixed_iters``: its
        measurement knob -- the checks never stop the loop)."""
        from .sinkhorn import _fp32_guard
        if max_iters < 1 or inner_iters < 1:
            raise ValueError("max_iters and inner_iters must be >= 1")
        if not (threshold > 0):
            raise ValueError("threshold must be positive")
        if fixed_iters:
            threshold = -1.0
        sched = eps if isinstance(eps, EpsilonSchedule) else EpsilonSchedule(float(eps))
        _fp32_guard(sched, inner_iters, max_iters)
        comm = self.comm
        if self.loop == "native":
            f_dev, g_dev, iters, conv, errs, duals = self._solve_native(
                sched, threshold, max_iters, inner_iters, g_init)
        else:
            eng = self.engine
            eng.reset_first_bad()
            which, iters, conv, errs, duals = sharded_loop(eng, comm, sched, threshold, max_iters,
                                                           inner_iters, g_init, p2p=self.p2p)
            f_dev, g_dev = eng.f_result(which).clone(), eng.g_result().clone()
        f_full = None
        if gather_f:
            import torch
            n_total, world = self.n_total, comm.world
            width = -(-n_total // world) + 1
            pad = torch.full((width,), float("nan"), dtype=torch.float32, device=f_dev.device)
            pad[: self.hi - self.lo] = f_dev
            allf = comm.all_gather_rows(pad).cpu().numpy().astype(np.float64)
            f_full = np.concatenate([allf[r, : shard_rows(n_total, world, r)[1]
                                           - shard_rows(n_total, world, r)[0]]
                                     for r in range(world)])
        return ShardedSinkhornOutput(
            f_local=f_dev.cpu().numpy().astype(np.float64), g=g_dev.cpu().numpy().astype(np.float64),
            errors=errs, dual_trace=duals, iterations=iters, converged=conv, eps=sched.target,
            row_offset=self.lo, n_total=self.n_total, f=f_full, f_device=f_dev, g_device=g_dev)


def solve_sinkhorn_sharded(x, y, eps, a=None, b=None, *, threshold: float = 1e-3,
                           max_iters: int = 2000, inner_iters: int = 10, g_init=None,
                           comm=None, x_is_local: bool = False, n_total: int | None = None,
                           impl: str = "auto", gather_f: bool = False,
                           cost_fn: str = "sqeucl", exchange: str = "auto",
                           fixed_iters: bool = False) -> ShardedSinkhornOutput:
    """Row-sharded ``solve_sinkhorn`` on a point cloud (one rank per GPU):
    ``ShardedProblem(x, y, a, b, ...).solve(eps, ...)``."""
    if max_iters < 1 or inner_iters < 1:
        raise ValueError("max_iters and inner_iters must be >= 1")
    if not (threshold > 0):
        raise ValueError("threshold must be positive")
    prob = ShardedProblem(x, y, a, b, comm=comm, x_is_local=x_is_local, n_total=n_total,
                          impl=impl, cost_fn=cost_fn, exchange=exchange)
    return prob.solve(eps, threshold=threshold, max_iters=max_iters, inner_iters=inner_iters,
                      g_init=g_init, gather_f=gather_f, fixed_iters=fixed_iters)


def _absmax(p) -> float:
    import torch
    amax = torch.empty(1, dtype=torch.float32, device=p.device)
    N.check(N.lib().otk_absmax(N.ptr(p), p.numel(), N.ptr(amax), stream()), "absmax")
    return float(amax.item())


def _dev_of(x):
    import torch
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return device()


def reg_ot_cost_sharded(out: ShardedSinkhornOutput, x_local, y, a_local, b, comm=None,
                        cost_fn: str = "sqeucl"):
    """reg_ot_cost (sinkhorn.py:210-216) over row shards: online local sums + rank-order total."""
    import torch
    from .geometry import _Cloud, centered_points, cost_fn_flags
    comm = comm or TorchComm()
    cflags = cost_fn_flags(cost_fn)
    cx, cy = (_Cloud(p) for p in centered_points(x_local, y, cost_fn))
    cx.prepare(1.0, False)
    cy.prepare(1.0, False)
    lib = N.lib()
    ws = torch.empty(lib.otk_cost_workspace_bytes(cx.n, cy.n), dtype=torch.uint8, device=cx.p.device)
    res = torch.zeros(2, dtype=torch.float64, device=cx.p.device)
    f_d = as_device_f32(out.f_device if out.f_device is not None else out.f_local)
    g_d = as_device_f32(out.g_device if out.g_device is not None else out.g)
    N.check(lib.otk_cost_partial(N.ptr(cx.p), N.ptr(cx.sq), cx.n, N.ptr(cy.p), N.ptr(cy.sq), cy.n,
                                 cx.d, N.ptr(f_d), N.ptr(g_d), float(out.eps), cflags, N.ptr(res),
                                 N.ptr(ws), stream()), "reg_ot_cost")
    a_local = np.asarray(a_local, dtype=float)
    b = np.asarray(b, dtype=float)
    with np.errstate(invalid="ignore"):
        fa = float(np.where(a_local > 0, out.f_local * a_local, 0.0).sum())
    loc = np.array([*res.cpu().numpy(), fa])
    rows = comm.all_gather_host(loc, cx.p.device)
    transport, mass, fa_tot = (float(sum(rows[r, k] for r in range(rows.shape[0]))) for k in range(3))
    with np.errstate(invalid="ignore"):
        gb = float(np.where(b > 0, out.g * b, 0.0).sum())
    from .sinkhorn import RegOTCost
    return RegOTCost(transport, fa_tot + gb - out.eps * (mass - 1.0))
