"""ctypes binding of libotk_sm100.so (the C ABI declared in include/otk.h).

The library is built in-tree by ``_build.build()`` for sm_100a.  There is no
CPU fallback: a missing library or a machine without a CUDA device raises.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

# OTK_LIB: an alternative build of the same ABI (A/B timing of kernel revisions)
_LIB_PATH = os.environ.get("OTK_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libotk_sm100.so")
_lib = None

OTK_OK, OTK_EINVAL, OTK_ECUDA, OTK_ENOTSUP, OTK_ENCCL = 0, -1, -2, -3, -4
OTK_DIVERGED, OTK_BAD_POTENTIAL = 1, 2
OTK_SAME_POINTS, OTK_CLAMP, OTK_IMPL_SIMT, OTK_IMPL_TC = 0x1, 0x2, 0x10, 0x20
OTK_IMPL_NOPERSIST = 0x40
OTK_ANCHOR_INIT, OTK_IMPL_NOANCHOR = 0x80, 0x100
OTK_COST_EUCL = 0x4
OTK_FIN_SOLVER, OTK_FIN_APPLY, OTK_FIN_LOG2 = 0, 1, 2
ABI_VERSION = 7

P = C.c_void_p
I64, I32, F32, F64, SZ = C.c_int64, C.c_int32, C.c_float, C.c_double, C.c_size_t


class SolveArgs(C.Structure):
    """Mirror of ``otk_solve_args`` (include/otk.h)."""

    _fields_ = [
        ("x", P), ("y", P), ("n", I64), ("m", I64), ("d", I32),
        ("a", P), ("b", P), ("log_a", P), ("log_b", P), ("same_points", I32),
        ("eps_target", F64), ("eps_init_scale", F64), ("eps_decay", F64),
        ("threshold", F64), ("max_iters", I32), ("inner_iters", I32),
        ("g_init", P), ("flags", I32), ("use_graphs", I32),
        ("f_out", P), ("g_out", P), ("errors", P), ("duals", P), ("max_checks", I32),
        ("n_checks", I32), ("iterations", I32), ("converged", I32), ("fail_iter", I32),
        ("launches", I32), ("workspace", P), ("workspace_bytes", SZ), ("stream", P),
        ("f_host", P), ("g_host", P),
    ]


class Exchange(C.Structure):
    """Mirror of ``otk_exchange`` (include/otk.h): multi-GPU exchange over peer memory."""

    _fields_ = [("local", P), ("world", I32), ("rank", I32), ("epoch", C.c_uint32)]


# name -> (restype, argtypes); every symbol declared in include/otk.h
SIGNATURES = {
    "otk_abi_version": (C.c_int, []),
    "otk_last_error": (C.c_char_p, []),
    "otk_device_query": (C.c_int, [C.c_int, P, P, P]),
    "otk_prep_points": (C.c_int, [P, I64, I32, P, P, P, P, P, I32, F32, P]),
    "otk_split_scale": (F32, [F32, I32]),
    "otk_absmax": (C.c_int, [P, I64, P, P]),
    "otk_points_flags": (C.c_int, [P, I64, P, I64, I32, I32, P, P]),
    "otk_mean_cost_pairs": (C.c_int, [P, P, P, P, I64, I32, I32, P, P]),
    "otk_column_median": (C.c_int, [P, I64, I32, P, P]),
    "otk_shift_points": (C.c_int, [P, I64, I32, P, P, P]),
    "otk_make_bias": (C.c_int, [P, I64, F32, P, P, I32, P]),
    "otk_lse_partial": (C.c_int, [P, P, P, P, P, I64, P, P, P, P, P, I64, I32, I32, F32, P, F32,
                                  I32, I32, P, P]),
    "otk_lse_suggest_nsplit": (C.c_int, [I64, I64, I32, I32]),
    "otk_lse_uses_tc": (C.c_int, [I32, I32]),
    "otk_lse_finalize": (C.c_int, [P, I32, I64, P, I32, F32, F32, P, P, P, I32, P]),
    "otk_lse_step_workspace_bytes": (SZ, [I64]),
    "otk_lse_step_anchored": (C.c_int, [I64, I64, I32, I32]),
    "otk_lse_step": (C.c_int, [P, P, P, P, P, I64, P, P, P, P, P, I64, I32, I32, F32, P, F32, I32,
                               I32, P, P, I32, F32, F32, P, P, P, I32, P, P, C.POINTER(Exchange), P]),
    "otk_exchange_bytes": (SZ, [I32, I64]),
    "otk_exchange_alloc": (C.c_int, [SZ, C.POINTER(P)]),
    "otk_exchange_free": (C.c_int, [P]),
    "otk_ipc_handle": (C.c_int, [P, P]),
    "otk_ipc_open": (C.c_int, [P, C.POINTER(P)]),
    "otk_ipc_close": (C.c_int, [P]),
    "otk_exchange_set_peers": (C.c_int, [P, I32, I64, P, P]),
    "otk_exchange_finalize": (C.c_int, [P, I32, I64, C.c_uint32, P, I32, F32, F32, P, P, P, I32,
                                        C.c_uint32, P]),
    "otk_exchange_status": (C.c_int, [P, P, P]),
    "otk_exchange_check": (C.c_int, [P, I32, I32, I64, P, P, P, C.c_uint32, P]),
    "otk_check_workspace_bytes": (SZ, []),
    "otk_check": (C.c_int, [P, P, P, I64, P, P, I64, F64, P, P, P]),
    "otk_cost_workspace_bytes": (SZ, [I64, I64]),
    "otk_cost_partial": (C.c_int, [P, P, I64, P, P, I64, I32, P, P, F64, I32, P, P, P]),
    "otk_transport_matrix": (C.c_int, [P, P, I64, P, P, I64, I32, P, P, F64, I32, P, P]),
    "otk_grad_points": (C.c_int, [P, P, I64, P, P, I64, I32, P, P, F64, I32, P, P]),
    "otk_dense_cost": (C.c_int, [P, P, I64, I64, I64, I32, I32, P, P, P]),
    "otk_dense_transpose": (C.c_int, [P, I64, I64, I64, P, P]),
    "otk_dense_lse": (C.c_int, [P, I64, I64, I64, I32, P, P, I32, P, P, P, P, P, P, I32, P]),
    "otk_check_batched": (C.c_int, [P, P, P, I64, P, P, I64, I64, P, P, P, P]),
    "otk_dense_plan": (C.c_int, [P, I64, I64, P, P, F64, P, P]),
    "otk_dense_solve_fits": (C.c_int, [I64, I64]),
    "otk_dense_cluster_plan": (C.c_int, [I64, I64, I64, P, P]),
    "otk_solve_dense_batched": (C.c_int, [P, I64, I64, I64, P, P, P, P, P, P, P, F64, I32, I32, I32,
                                          P, P, P, P, P, I32, P]),
    "otk_dense_cost_reduce": (C.c_int, [P, I64, I64, I64, P, P, P, P, P]),
    "otk_bench_pipes": (C.c_int, [P, P, P]),
    "otk_bench_read": (C.c_int, [P, I64, P, P]),
    "otk_bench_smem": (C.c_int, [P, P]),
    "otk_barycenter_ld": (I64, [I64]),
    "otk_barycenter_part_len": (I64, [I64, I32]),
    "otk_barycenter_pad": (C.c_int, [P, I64, I64, P, P, P]),
    "otk_solve_barycenter": (C.c_int, [P, P, I64, I64, I32, P, P, F64, F64, I32, P, P, P, P, P, P,
                                       P, P]),
    "otk_solve_workspace_bytes": (SZ, [C.POINTER(SolveArgs)]),
    "otk_solve_pointcloud": (C.c_int, [C.POINTER(SolveArgs)]),
    "otk_solve_pointcloud_sharded": (C.c_int, [C.POINTER(SolveArgs), C.POINTER(Exchange), F32,
                                               C.c_uint32]),
}


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load the CUDA library (loudly failing if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(
                f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        if not os.environ.get("OTK_LIB"):
            from . import _build
            stale = _build.stale_reason()
            if stale:
                raise RuntimeError(f"{_LIB_PATH} is stale ({stale}): rebuild it with "
                                   "`python -c 'import __graft_entry__ as g; g.build()'`")
        handle = C.CDLL(_LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.otk_abi_version() != ABI_VERSION:
            raise RuntimeError("libotk_sm100.so ABI version mismatch; rebuild")
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().otk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> int:
    """Map a negative status to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == OTK_EINVAL:
        raise ValueError(msg)
    if rc == OTK_ENOTSUP:
        raise NotImplementedError(msg)
    raise errors.OtkitError(msg) if rc == OTK_ENCCL else RuntimeError(msg)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()
