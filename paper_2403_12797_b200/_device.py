"""Device-memory plumbing on top of torch (allocation, host<->device copies, streams).

torch is used only as an allocator / stream provider here; all arithmetic on the posterior
path happens in libfagp_b200.so.
"""

from __future__ import annotations

import numpy as np

_DTYPES = {"float64": "float64", "int64": "int64", "int32": "int32", "uint8": "uint8"}


def _torch():
    import torch

    return torch


def device_of(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        from ._lib import ExtensionMissing

        raise ExtensionMissing("no CUDA device: paper_2403_12797_b200 runs only on the GPU (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def empty(shape, dtype="float64", device=None):
    torch = _torch()
    return torch.empty(shape, dtype=getattr(torch, _DTYPES[dtype]), device=device_of(device))


def zeros(shape, dtype="float64", device=None):
    torch = _torch()
    return torch.zeros(shape, dtype=getattr(torch, _DTYPES[dtype]), device=device_of(device))


def to_device(a, device=None, dtype="float64"):
    """numpy / list / torch tensor -> contiguous CUDA float64 tensor (no copy when already so)."""
    torch = _torch()
    tdt = getattr(torch, _DTYPES[dtype])
    dev = device_of(device)
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=tdt)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.dtype(dtype)))
    return torch.from_numpy(arr).to(dev, non_blocking=False)


def to_host(t):
    """CUDA tensor -> numpy.  Large results land in page-locked memory from torch's pinned
    caching allocator (DMA at full link speed, no first-touch page faults); the returned array
    keeps that buffer alive, and it returns to the cache when the array is dropped."""
    torch = _torch()
    t = t.detach()
    if not t.is_cuda or t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()


def upload_async(a, device=None):
    """Start the H2D copy of a host tensor/array on a side stream; returns (device tensor,
    event).  Pinned sources copy asynchronously; the caller waits on the event."""
    torch = _torch()
    dev = device_of(device)
    if isinstance(a, torch.Tensor) and a.is_cuda:
        return to_device(a, dev), None
    main = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        if isinstance(a, torch.Tensor):
            src = a.to(dtype=torch.float64).contiguous()
        else:
            src = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
        d = src.to(dev, non_blocking=src.is_pinned())
        ev = torch.cuda.Event()
        ev.record(side)
    d.record_stream(main)
    return d, ev


def wait_upload(ev):
    """Make the current stream wait for an upload_async event (None: nothing pending)."""
    if ev is not None:
        _torch().cuda.current_stream().wait_event(ev)


def is_tensor(a):
    torch = _torch()
    return isinstance(a, torch.Tensor)


def points_shape(X, p, name):
    """Validate an (N, p) point set's shape without copying it (posterior.py:93-97)."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        shape = tuple(X.shape) if X.dim() == 2 else ((1, X.shape[0]) if X.dim() == 1 and X.numel() else (0, p))
    else:
        shape = np.atleast_2d(np.asarray(X, dtype=float)).shape
    if len(shape) != 2 or shape[1] != p:
        raise ValueError(f"{name} has {shape[-1]} columns, expected p={p}")


def points(X, p, name):
    """Coerce an (N, p) point set to a device tensor, mirroring posterior._as_points
    (posterior.py:93-97) and the host-side checks of eigensystem (mercer.py:331-335)."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        Xt = X
        if Xt.dim() == 1:
            Xt = Xt.reshape(1, -1) if Xt.numel() else Xt.reshape(0, p)
        if Xt.dim() != 2 or Xt.shape[1] != p:
            raise ValueError(f"{name} has {Xt.shape[-1]} columns, expected p={p}")
        return to_device(Xt)
    Xh = np.atleast_2d(np.asarray(X, dtype=float))
    if Xh.shape[1] != p:
        raise ValueError(f"{name} has {Xh.shape[1]} columns, expected p={p}")
    # finiteness is checked on the device (FAGP_FLAG_X_NONFINITE from fagp_basis_eval)
    return to_device(Xh)


def is_cuda(a):
    torch = _torch()
    return isinstance(a, torch.Tensor) and a.is_cuda


def host_points(X, p, name):
    """Validate an (N, p) HOST point set like :func:`points` without uploading it; returns a
    contiguous float64 numpy array or CPU tensor (pinned tensors stay pinned)."""
    torch = _torch()
    if isinstance(X, torch.Tensor):
        Xt = X.detach()
        if Xt.dim() == 1:
            Xt = Xt.reshape(1, -1) if Xt.numel() else Xt.reshape(0, p)
        if Xt.dim() != 2 or Xt.shape[1] != p:
            raise ValueError(f"{name} has {Xt.shape[-1]} columns, expected p={p}")
        if Xt.dtype != torch.float64 or not Xt.is_contiguous():
            Xt = Xt.to(torch.float64).contiguous()
        return Xt
    Xh = np.atleast_2d(np.asarray(X, dtype=float))
    if Xh.shape[1] != p:
        raise ValueError(f"{name} has {Xh.shape[1]} columns, expected p={p}")
    return np.ascontiguousarray(Xh)


def host_vector(y, N, name="y"):
    """Validate a HOST (N,) vector without uploading it."""
    torch = _torch()
    if isinstance(y, torch.Tensor):
        yt = y.detach()
        if tuple(yt.shape) != (N,):
            raise ValueError(f"{name} has shape {tuple(yt.shape)}, expected ({N},)")
        return yt.to(torch.float64).contiguous() if yt.dtype != torch.float64 or not yt.is_contiguous() else yt
    yh = np.asarray(y, dtype=float)
    if yh.shape != (N,):
        raise ValueError(f"{name} has shape {yh.shape}, expected ({N},)")
    return np.ascontiguousarray(yh)
