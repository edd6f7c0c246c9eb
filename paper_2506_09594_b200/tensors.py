"""Host <-> device layout plumbing.

The reference stores tensors column-major (first index fastest,
tenrec/core.py:1-8) and every kernel of this package reads that layout.  A
``ColMajor`` wraps a flat CUDA buffer plus its dims; numpy inputs are copied
(pinned host -> HBM) in Fortran order, torch CUDA inputs are permuted once.
Results go back in the caller's container type.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib


class ColMajor:
    __slots__ = ("flat", "dims", "kind", "np_dtype")

    def __init__(self, flat, dims, kind, np_dtype):
        self.flat = flat
        self.dims = tuple(int(v) for v in dims)
        self.kind = kind  # "numpy" | "torch"
        self.np_dtype = np_dtype

    @property
    def dtype_code(self):
        import torch

        return _lib.F32 if self.flat.dtype == torch.float32 else _lib.F64

    @property
    def ptr(self):
        return self.flat.data_ptr()

    def numel(self):
        return int(math.prod(self.dims))


def _torch():
    import torch

    return torch


def _upload(a: np.ndarray):
    """Flat column-major CUDA copy of a numpy array.

    F-ordered arrays go up as they are; anything else goes up in C order (one
    contiguous host pass at most) and is transposed on the device -- a host
    ``ravel(order="F")`` of a C-ordered array is a strided gather that costs
    seconds at these sizes.  The host side goes through torch's cached
    page-locked buffers so the DMA runs at full PCIe/C2C speed.
    """
    torch = _torch()
    fortran = a.flags.f_contiguous
    if not fortran:
        a = np.ascontiguousarray(a)
    raw = a.view(np.uint8) if a.dtype == np.bool_ else a
    host = torch.from_numpy(raw.ravel(order="F" if fortran else "C"))
    if host.numel():
        dev = host.pin_memory().to("cuda", non_blocking=True)
    else:
        dev = host.to("cuda")
    if not fortran and a.ndim > 1:
        dev = dev.reshape(a.shape).permute(*reversed(range(a.ndim))).contiguous().reshape(-1)
    return dev


def to_device(x, dtype=None) -> ColMajor:
    """Column-major CUDA copy of ``x`` (numpy array, scalar list or torch tensor)."""
    torch = _torch()
    _lib.lib()
    if isinstance(x, torch.Tensor):
        if dtype is None:
            dtype = torch.float32 if x.dtype == torch.float32 else torch.float64
        dims = tuple(x.shape)
        t = x.to(device="cuda", dtype=dtype)
        flat = t.permute(*reversed(range(t.dim()))).contiguous().reshape(-1) if t.dim() else t
        return ColMajor(flat, dims, "torch", None)
    a = np.asarray(x)
    if dtype is None:
        np_dtype = np.float32 if a.dtype == np.float32 else np.float64
    else:
        np_dtype = np.float32 if dtype == torch.float32 else np.float64
    a = a.astype(np_dtype, copy=False)
    return ColMajor(_upload(a), a.shape, "numpy", np_dtype)


def mask_to_device(mask):
    """Observation mask as a flat column-major uint8 CUDA buffer."""
    torch = _torch()
    if isinstance(mask, torch.Tensor):
        m = mask.to(device="cuda", dtype=torch.uint8)
        return m.permute(*reversed(range(m.dim()))).contiguous().reshape(-1)
    return _upload(np.asarray(mask, dtype=bool))


def empty_like(cm: ColMajor, dims=None) -> ColMajor:
    torch = _torch()
    dims = cm.dims if dims is None else tuple(dims)
    flat = torch.empty(int(math.prod(dims)), dtype=cm.flat.dtype, device="cuda")
    return ColMajor(flat, dims, cm.kind, cm.np_dtype)


def from_device(cm: ColMajor):
    """Back to the caller's container: numpy (same dtype) or a CUDA tensor view.

    numpy results are returned in page-locked memory from torch's caching host
    allocator (one DMA, no extra host copy; the block is recycled once the
    array is dropped).
    """
    torch = _torch()
    if cm.kind == "numpy":
        if cm.flat.numel() == 0:
            return np.zeros(cm.dims, dtype=cm.np_dtype, order="F")
        host = torch.empty(cm.flat.numel(), dtype=cm.flat.dtype, pin_memory=True)
        host.copy_(cm.flat, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host.numpy().reshape(cm.dims, order="F")
    d = len(cm.dims)
    return cm.flat.reshape(tuple(reversed(cm.dims))).permute(*reversed(range(d)))


_WORKSPACES = {}


def workspace(nbytes: int):
    """Cached device workspace of at least ``nbytes`` (per device and host thread:
    concurrent host threads never share one)."""
    import threading

    torch = _torch()
    key = (torch.cuda.current_device(), threading.get_ident())
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
        _WORKSPACES[key] = buf
    return buf
