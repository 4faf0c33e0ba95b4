"""Device plumbing: CUDA device/stream from torch, host<->device conversion.

torch is used only for device memory, streams and (multi-GPU) the process
group; every computation on the Sinkhorn path is a kernel of libotk_sm100.so.
"""

from __future__ import annotations

import numpy as np


def is_torch(v) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor)


def device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_12324_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def as_device_f32(v, async_pinned: bool = False):
    """numpy / torch -> contiguous float32 CUDA tensor (no copy if already one).
    ``async_pinned``: copy pinned host tensors asynchronously on the current
    stream -- only for callers that synchronise before returning to the user
    (the geometry's validation reads back a flag right after)."""
    import torch
    dev = device()
    if is_torch(v):
        if v.device.type == "cuda" and v.dtype == torch.float32 and v.is_contiguous():
            return v
        nb = async_pinned and v.device.type == "cpu" and v.is_pinned()
        return v.to(device=dev, dtype=torch.float32, non_blocking=nb).contiguous()
    arr = np.ascontiguousarray(np.asarray(v), dtype=np.float32)
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def to_output(t, like):
    """Return a device result in the caller's convention: torch in -> torch out,
    numpy in -> float64 numpy out (the reference returns float64 ndarrays)."""
    if is_torch(like):
        return t
    return t.cpu().numpy().astype(np.float64)


def validate_potential(p, size, name):
    """geometry.py:65-72: shape (size,), -inf allowed, NaN / +inf rejected.
    Returns a float32 CUDA tensor."""
    import torch
    if is_torch(p):
        if tuple(p.shape) != (size,):
            raise ValueError(f"{name} must have shape ({size},), got {tuple(p.shape)}")
        bad = torch.isnan(p).any() | (p == float("inf")).any()
        if bool(bad.item()):
            raise ValueError(f"{name} contains NaN or +inf entries")
        return as_device_f32(p)
    p = np.asarray(p, dtype=float)
    if p.shape != (size,):
        raise ValueError(f"{name} must have shape ({size},), got {p.shape}")
    if np.isnan(p).any() or np.any(p == np.inf):
        raise ValueError(f"{name} contains NaN or +inf entries")
    return as_device_f32(p)


class nvtx_range:
    """NVTX range around host-driven device work (the C++ loops carry their own,
    csrc/solve.cu); a no-op where NVTX is unavailable."""

    def __init__(self, name: str):
        self.name = name
        self.on = False

    def __enter__(self):
        try:
            import torch
            torch.cuda.nvtx.range_push(self.name)
            self.on = True
        except Exception:  # noqa: BLE001 -- profiling aid only
            pass
        return self

    def __exit__(self, *exc):
        if self.on:
            import torch
            torch.cuda.nvtx.range_pop()
