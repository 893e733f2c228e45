"""Device-buffer helpers: column-major FP64 matrices held in PyTorch.

An m x n matrix lives on the device as a contiguous torch tensor of shape
(n, m) -- row c is column c -- i.e. column-major storage, the layout the
reference (and the paper) uses.  Host numpy arrays come
in and go out in Fortran order, like the reference's.
"""

from __future__ import annotations

import numpy as np
import torch


def device() -> torch.device:
    from . import _lib

    _lib.require_cuda()  # loud NativeUnavailable without a B200 / the library
    return torch.device("cuda", torch.cuda.current_device())


def is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


def out_mode(a) -> str:
    """How results are returned for input `a`: 'numpy', 'device' (CUDA
    tensors) or 'host' (CPU torch tensors, pinned when large)."""
    if not is_torch(a):
        return "numpy"
    return "device" if a.is_cuda else "host"


def to_colmajor(a, copy: bool = False) -> torch.Tensor:
    """m x n host or device matrix -> (n, m) contiguous FP64 device tensor."""
    if is_torch(a):
        t = a.to(device=device(), dtype=torch.float64)
        if t.ndim != 2:
            raise ValueError("expected a 2-d matrix")
        st = t.t()
        if st.is_contiguous() and not copy and st.data_ptr() == a.data_ptr():
            return st
        return st.contiguous() if not copy else st.contiguous().clone()
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("expected a 2-d matrix")
    hc = np.ascontiguousarray(arr.T)
    if not hc.flags.writeable:  # e.g. np.frombuffer data: torch wants writable memory
        hc = hc.copy()
    host = torch.from_numpy(hc)
    if host.numel() >= (1 << 20):
        host = host.pin_memory()
    return host.to(device(), non_blocking=True)


def _to_host(t: torch.Tensor) -> torch.Tensor:
    if t.numel() >= (1 << 20):
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return t.cpu()


def from_colmajor(t: torch.Tensor, mode):
    """(n, m) column-major storage -> m x n result: numpy F-order array
    ('numpy' / True), CUDA tensor view ('device' / False) or CPU tensor
    view ('host')."""
    if mode is True or mode == "numpy":
        return np.asfortranarray(_to_host(t).numpy().T)
    if mode == "host":
        return _to_host(t).t()
    return t.t()


def vector_out(t: torch.Tensor, mode):
    if mode is True or mode == "numpy":
        return t.cpu().numpy()
    if mode == "host":
        return t.cpu()
    return t
