"""Circulant difference operators and the FFT-diagonalised gradient solve.

Mirrors ``tenrec.gradient`` (gradient.py:1-106): ``GradientSet(dims, modes)``
validates the smoothness directions exactly as gradient.py:55-67 does, and
``solve_grad_system(b, grads, gset)`` returns
``(I + sum_k D_k^T D_k)^{-1} (b + sum_k D_k^T grads[k])``.  The solve runs on
the device through ``tr_gradsys_*``: one real-to-half-spectrum pass, one
complex pass per further axis with the diagonal division fused into the last
one, and the inverse passes.  The plan (twiddles, eigenvalue tables, spectrum
buffer) is built on first use per dtype and cached on the GradientSet.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .tensors import empty_like, from_device, to_device

__all__ = ["GradientSet", "solve_grad_system"]


class GradientSet:
    """Smoothness directions of a tensor shape (gradient.py:44-67)."""

    def __init__(self, dims, modes):
        self.dims = tuple(int(n) for n in dims)
        self.modes = tuple(int(k) for k in modes)
        if not self.modes:
            raise ValueError("gradient mode set must be nonempty")
        for k in self.modes:
            if not 0 <= k < len(self.dims):
                raise ValueError(f"gradient mode {k} out of range for dims {self.dims}")
        self._plans = {}

    def __repr__(self):
        return f"GradientSet(dims={self.dims}, modes={self.modes})"

    @property
    def denominator(self) -> np.ndarray:
        """``1 + sum_k 4 sin^2(pi j_k / n_k)`` (gradient.py:63-67, 75-80), host-side."""
        denom = np.ones(self.dims)
        for k in self.modes:
            n = self.dims[k]
            shape = [1] * len(self.dims)
            shape[k] = n
            denom = denom + (4.0 * np.sin(np.pi * np.arange(n) / n) ** 2).reshape(shape)
        return denom

    def _plan(self, dtype_code: int):
        h = self._plans.get(dtype_code)
        if h is None:
            lib = _lib.lib()
            uniq = []
            for k in self.modes:
                if k not in uniq:
                    uniq.append(k)
            dims = (ctypes.c_int64 * len(self.dims))(*self.dims)
            modes = (ctypes.c_int * len(uniq))(*uniq)
            hp = ctypes.c_void_p()
            _lib.check(lib.tr_gradsys_create(dtype_code, len(self.dims), dims, len(uniq), modes,
                                             ctypes.byref(hp)))
            h = (hp.value, tuple(uniq))
            self._plans[dtype_code] = h
        return h

    def __del__(self):
        lib = _lib._LIB
        if lib is None:
            return
        for h, _ in getattr(self, "_plans", {}).values():
            try:
                lib.tr_gradsys_destroy(h)
            except Exception:  # interpreter shutdown
                pass


def solve_grad_system(b, grads: dict, gset: GradientSet):
    """``(I + sum_k D_k^T D_k)(L) = b + sum_k D_k^T(grads[k])`` (gradient.py:90-106).

    ``b`` and every ``grads[k]`` are numpy arrays or torch tensors of shape
    ``gset.dims``; the result comes back in ``b``'s container (numpy float64
    for numpy input as in the reference, or a CUDA tensor of ``b``'s dtype).
    """
    import torch

    bshape = tuple(b.shape)
    if bshape != gset.dims:
        raise ValueError(f"rhs shape {bshape} does not match gradient set {gset.dims}")
    dtype = b.dtype if isinstance(b, torch.Tensor) and b.dtype in (torch.float32,
                                                                    torch.float64) else torch.float64
    bd = to_device(b, dtype)
    h, uniq = gset._plan(bd.dtype_code)
    gd = []
    for k in uniq:
        g = grads[k]
        if tuple(g.shape) != bshape:
            raise ValueError(f"gradient term for mode {k} has shape {tuple(g.shape)}")
        gd.append(to_device(g, dtype))
    # a mode listed twice contributes its term twice (gradient.py:100-104)
    mult = {k: gset.modes.count(k) for k in uniq}
    if any(m > 1 for m in mult.values()):
        raise ValueError("repeated gradient modes are not supported by the device plan")
    out = empty_like(bd)
    ptrs = (ctypes.c_void_p * len(gd))(*[g.ptr for g in gd])
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().tr_gradsys_solve(h, bd.ptr, ptrs, out.ptr, ctypes.c_void_p(stream)))
    res = from_device(out)
    if bd.kind == "numpy":
        return np.asarray(res, dtype=np.float64)
    return res
