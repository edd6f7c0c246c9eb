"""The seven nonconvex penalties, mirroring tenrec/penalties.py.

Same class names, parameters, defaults and validation errors as the
reference.  ``prox`` runs the CUDA kernel ``tr_prox`` (csrc/prox.cuh) on the
device; numpy / scalar inputs are copied over and back so the call is a
drop-in.  ``value`` is a monitoring helper (never on the hot path) evaluated
with torch elementwise ops on the input's device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

PENALTY_NAMES = ("l1", "firm", "mcp", "scad", "lq", "capped-lq", "log")


class Penalty:
    kind: int = -1

    def params(self):
        return 0.0, 0.0

    def encode(self):
        """(kind, p0, p1) -- the C ABI's penalty encoding."""
        p0, p1 = self.params()
        return self.kind, float(p0), float(p1)

    def prox(self, mu, v):
        """Global minimiser of value(|x|, mu) + (x - v)^2 / 2, on the GPU."""
        import torch

        if mu < 0:
            raise ValueError("prox level mu must be >= 0")
        lib = _lib.lib()
        kind, p0, p1 = self.encode()
        if isinstance(v, torch.Tensor):
            src = v.to(device="cuda")
            if src.dtype not in (torch.float32, torch.float64):
                src = src.double()
            src = src.contiguous()
            out = torch.empty_like(src)
            code = _lib.F32 if src.dtype == torch.float32 else _lib.F64
            _lib.check(lib.tr_prox(code, kind, p0, p1, float(mu), ctypes.c_void_p(src.data_ptr()),
                                   ctypes.c_void_p(out.data_ptr()), src.numel(),
                                   _lib.stream_ptr()))
            return out
        arr = np.asarray(v, dtype=np.float64)
        scalar = arr.ndim == 0
        dev = torch.from_numpy(np.ascontiguousarray(np.atleast_1d(arr))).to("cuda")
        out = torch.empty_like(dev)
        _lib.check(lib.tr_prox(_lib.F64, kind, p0, p1, float(mu), ctypes.c_void_p(dev.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()), dev.numel(), _lib.stream_ptr()))
        res = out.cpu().numpy().reshape(np.atleast_1d(arr).shape)
        return float(res[0]) if scalar else res

    def value(self, t, mu):
        import torch

        is_np = not isinstance(t, torch.Tensor)
        tt = torch.as_tensor(np.asarray(t, dtype=np.float64) if is_np else t)
        out = self._value(tt, float(mu), torch)
        return out.numpy() if is_np else out

    def objective(self, x, mu, v):
        return self.value(np.abs(x), mu) + 0.5 * (np.asarray(x) - v) ** 2

    def _value(self, t, mu, torch):
        raise NotImplementedError


@dataclass(frozen=True)
class L1(Penalty):
    kind = 0

    def _value(self, t, mu, torch):
        return mu * t


class _MinimaxConcave(Penalty):
    def params(self):
        return self.gamma, 0.0

    def _value(self, t, mu, torch):
        g = self.gamma
        return torch.where(t <= g * mu, mu * t - t ** 2 / (2.0 * g),
                           torch.full_like(t, g * mu ** 2 / 2.0))


@dataclass(frozen=True)
class MCP(_MinimaxConcave):
    gamma: float = 2.5
    kind = 2

    def __post_init__(self):
        if self.gamma <= 1:
            raise ValueError("MCP requires gamma > 1")


@dataclass(frozen=True)
class Firm(_MinimaxConcave):
    gamma: float = 2.5
    kind = 1

    def __post_init__(self):
        if self.gamma <= 1:
            raise ValueError("firm shrinkage requires gamma > 1")


@dataclass(frozen=True)
class SCAD(Penalty):
    a: float = 3.7
    kind = 3

    def __post_init__(self):
        if self.a <= 2:
            raise ValueError("SCAD requires a > 2")

    def params(self):
        return self.a, 0.0

    def _value(self, t, mu, torch):
        a = self.a
        quad = (2.0 * a * mu * t - t ** 2 - mu ** 2) / (2.0 * (a - 1.0))
        cap = torch.full_like(t, mu ** 2 * (a + 1.0) / 2.0)
        return torch.where(t <= mu, mu * t, torch.where(t <= a * mu, quad, cap))


@dataclass(frozen=True)
class Lq(Penalty):
    q: float = 0.5
    newton_iters: int = 50
    newton_tol: float = 1e-12
    kind = 4

    def __post_init__(self):
        if not 0 < self.q <= 1:
            raise ValueError("Lq requires q in (0, 1]")

    def params(self):
        return self.q, 0.0

    def threshold(self, mu):
        q = self.q
        if q == 1.0:
            return mu
        xh = (2.0 * mu * (1.0 - q)) ** (1.0 / (2.0 - q))
        return xh + mu * q * xh ** (q - 1.0)

    def _value(self, t, mu, torch):
        return mu * t ** self.q


@dataclass(frozen=True)
class CappedLq(Penalty):
    q: float = 0.5
    theta: float = 1.0
    kind = 5

    def __post_init__(self):
        if not 0 < self.q <= 1:
            raise ValueError("capped Lq requires q in (0, 1]")
        if self.theta <= 0:
            raise ValueError("capped Lq requires theta > 0")

    def params(self):
        return self.q, self.theta

    def _value(self, t, mu, torch):
        return mu * torch.clamp(t, max=self.theta) ** self.q


@dataclass(frozen=True)
class LogPenalty(Penalty):
    gamma: float = 1.0
    kind = 6

    def __post_init__(self):
        if self.gamma <= 0:
            raise ValueError("log penalty requires gamma > 0")

    def params(self):
        return self.gamma, 0.0

    def _value(self, t, mu, torch):
        return mu * torch.log1p(t / self.gamma)


def make_penalty(name: str, **params) -> Penalty:
    key = name.lower().replace("_", "-")
    table = {"l1": L1, "firm": Firm, "mcp": MCP, "scad": SCAD, "lq": Lq, "capped-lq": CappedLq,
             "log": LogPenalty}
    if key not in table:
        raise ValueError(f"unknown penalty {name!r}; choose from {PENALTY_NAMES}")
    return table[key](**params)


def encode(pen) -> tuple:
    """Encode this package's penalties or the reference's (same class names)."""
    if isinstance(pen, Penalty):
        return pen.encode()
    name = type(pen).__name__
    fields = {"L1": (0, 0.0, 0.0), "Firm": (1, "gamma", None), "MCP": (2, "gamma", None),
              "SCAD": (3, "a", None), "Lq": (4, "q", None), "CappedLq": (5, "q", "theta"),
              "LogPenalty": (6, "gamma", None)}
    if name not in fields:
        raise TypeError(f"unsupported penalty object {pen!r}")
    kind, f0, f1 = fields[name]
    p0 = float(getattr(pen, f0)) if isinstance(f0, str) else 0.0
    p1 = float(getattr(pen, f1)) if isinstance(f1, str) else 0.0
    return kind, p0, p1
