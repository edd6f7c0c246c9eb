"""Trailing-mode transform specification, mirroring tenrec/transform.py:40-105.

Only the description lives on the host (kind, explicit matrices, scalings and
their validation).  The transform itself runs on the device as a chain of
complex mode products (csrc/core_svt.cuh: k_build_transform, k_mode_product).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class TransformError(ValueError):
    """Transform construction or application failure."""


@dataclass(frozen=True)
class Transform:
    kind: str = "fft"
    matrices: tuple = field(default=None)
    alphas: tuple = field(default=None)

    @classmethod
    def fft(cls) -> "Transform":
        return cls(kind="fft")

    @classmethod
    def dct(cls) -> "Transform":
        return cls(kind="dct")

    @classmethod
    def explicit(cls, matrices) -> "Transform":
        mats = tuple(np.asarray(m) for m in matrices)
        alphas = []
        for m in mats:
            if m.ndim != 2 or m.shape[0] != m.shape[1]:
                raise TransformError("explicit transform matrices must be square")
            n = m.shape[0]
            gram = m @ m.conj().T
            alpha = float(np.real(np.trace(gram)) / n)
            if alpha <= 0:
                raise TransformError("transform matrix has nonpositive scaling")
            if np.max(np.abs(gram - alpha * np.eye(n))) > 1e-10 * max(1.0, alpha):
                raise TransformError("matrix is not unitary up to scaling")
            alphas.append(alpha)
        return cls(kind="explicit", matrices=mats, alphas=tuple(alphas))

    def rho(self, shape) -> float:
        trailing = tuple(shape[2:])
        if self.kind == "fft":
            return float(np.prod(trailing)) if trailing else 1.0
        if self.kind == "dct":
            return 1.0
        self.check_shape(shape)
        return float(np.prod(self.alphas))

    def check_shape(self, shape):
        if self.kind != "explicit":
            return
        trailing = tuple(shape[2:])
        if len(trailing) != len(self.matrices):
            raise TransformError(f"transform built for {len(self.matrices)} trailing modes, "
                                 f"tensor has {len(trailing)}")
        for n, m in zip(trailing, self.matrices):
            if m.shape[0] != n:
                raise TransformError(f"transform matrix size {m.shape[0]} does not match "
                                     f"mode length {n}")

    def device_args(self, shape):
        """(kind code, device matrices pointer, host alphas, keepalive) for the C ABI."""
        import torch

        code = _lib.TRANSFORM_KINDS[self.kind]
        if self.kind != "explicit":
            return code, None, None, None
        self.check_shape(shape)
        flat = np.concatenate([np.asarray(m, dtype=np.complex128).ravel(order="C")
                               for m in self.matrices])
        dev = torch.from_numpy(flat.view(np.float64).copy()).to("cuda")
        alphas = (ctypes.c_double * len(self.alphas))(*self.alphas)
        return code, ctypes.c_void_p(dev.data_ptr()), alphas, dev


DEFAULT_TRANSFORM = Transform.fft()


def as_transform(t) -> Transform:
    """Accept this package's Transform or the reference's (same fields)."""
    if isinstance(t, Transform):
        return t
    kind = getattr(t, "kind", None)
    if kind == "explicit":
        return Transform.explicit(t.matrices)
    if kind in ("fft", "dct"):
        return Transform(kind=kind)
    raise TypeError(f"unsupported transform {t!r}")
