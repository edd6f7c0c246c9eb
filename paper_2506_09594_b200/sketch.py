"""Randomized Tucker sketching and the randomized t-SVT on the B200.

Drop-in for tenrec/sketch.py's fixed-rank path:
  SketchConfig          sketch.py:64-126 (same fields, defaults and errors)
  TuckerFactors         sketch.py:39-61
  rsthosvd_bki          sketch.py:211-270  -> C ABI tr_rsthosvd_bki
  gnhtsvt_randomized    sketch.py:430-456  -> C ABI tr_gnhtsvt_randomized

Sketch matrices come from the counter-based Philox stream (entry (c, t) of
processing step p is N(0,1) at (seed, p, c*b + t)), so results are
deterministic per seed and identical to the oracle fed the same stream.
``sketch_override=(g0, g1)`` replays externally drawn matrices instead.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .penalties import encode as encode_penalty
from .tensors import ColMajor, empty_like, from_device, to_device, workspace
from .transform import DEFAULT_TRANSFORM, as_transform


@dataclass
class TuckerFactors:
    core: object
    factors: list
    dims: tuple

    def reconstruct(self):
        import torch

        core = torch.as_tensor(self.core)
        if any(n == 0 for n in core.shape):
            return np.zeros(self.dims)
        out = core
        for mode, f in enumerate(self.factors):
            if f is not None:
                f = torch.as_tensor(f, device=out.device, dtype=out.dtype)
                out = torch.movedim(torch.tensordot(f, out, dims=([1], [mode])), 0, mode)
        return out.cpu().numpy() if isinstance(self.core, np.ndarray) else out

    @property
    def ranks(self) -> tuple:
        return tuple(f.shape[1] if f is not None else n for f, n in zip(self.factors, self.dims))


@dataclass
class SketchConfig:
    mode: str = "fixed-rank"
    order: tuple = None
    ranks: tuple = None
    blocks: tuple = None
    krylov: tuple = None
    eps: float = 0.05
    block: int = 10
    defl_tol: float = None
    seed: int = 0

    def validate(self, dims) -> None:
        d = len(dims)
        order = self.resolved_order(dims)
        for k in order:
            if not 0 <= k < d:
                raise ValueError(f"processing order entry {k} out of range")
        if self.mode == "fixed-rank":
            if self.ranks is None:
                raise ValueError("fixed-rank sketching requires target ranks")
            ranks, blocks, krylov = self.resolved_fixed_rank(order)
            for k, r, b, q in zip(order, ranks, blocks, krylov):
                if r > dims[k]:
                    raise ValueError(f"rank {r} exceeds mode-{k} length {dims[k]}")
                if not 1 <= b <= r:
                    raise ValueError(f"block size {b} must satisfy 1 <= b <= r ({r})")
                if (q + 1) * b < r:
                    raise ValueError(f"(q+1)*b = {(q + 1) * b} < rank {r} on mode {k}")
        elif self.mode == "fixed-accuracy":
            if not 0 < self.eps < 1:
                raise ValueError("eps must lie in (0, 1)")
            if self.block < 1:
                raise ValueError("block size must be >= 1")
            if self.defl_tol is not None and self.defl_tol <= 0:
                raise ValueError("deflation tolerance must be > 0")
        else:
            raise ValueError(f"unknown sketch mode {self.mode!r}")

    def resolved_order(self, dims) -> tuple:
        if self.order is not None:
            return tuple(int(k) for k in self.order)
        return tuple(range(len(dims)))

    def resolved_fixed_rank(self, order):
        ranks = self._per_order(self.ranks, order, "ranks")
        blocks = (self._per_order(self.blocks, order, "blocks") if self.blocks
                  else [max(1, int(np.ceil(r / 4))) for r in ranks])
        krylov = (self._per_order(self.krylov, order, "krylov") if self.krylov is not None
                  else [4] * len(order))
        return [int(v) for v in ranks], [int(v) for v in blocks], [int(v) for v in krylov]

    @staticmethod
    def _per_order(values, order, name):
        vals = list(values)
        if len(vals) != len(order):
            raise ValueError(f"{name} must provide one entry per processed mode")
        return vals


def _gpu_order_check(order):
    if tuple(order) != (0, 1):
        raise NotImplementedError(
            f"the B200 path compresses modes (0, 1) (the gnhtsvt_randomized default); "
            f"order {tuple(order)} is not supported yet")


def _override_ptrs(override, cm: ColMajor):
    if override is None:
        return None, None, ()
    import torch

    keep = []
    ptrs = []
    for g in override:
        t = torch.as_tensor(np.ascontiguousarray(g) if isinstance(g, np.ndarray) else g)
        t = t.to(device="cuda", dtype=cm.flat.dtype).contiguous()
        keep.append(t)
        ptrs.append(ctypes.c_void_p(t.data_ptr()))
    return ptrs[0], ptrs[1], keep


def _resolve(sketch: SketchConfig, dims):
    if sketch.order is None:
        sketch = SketchConfig(mode=sketch.mode, order=(0, 1), ranks=sketch.ranks,
                              blocks=sketch.blocks, krylov=sketch.krylov, eps=sketch.eps,
                              block=sketch.block, defl_tol=sketch.defl_tol, seed=sketch.seed)
    sketch.validate(dims)
    if sketch.mode != "fixed-rank":
        raise NotImplementedError("fixed-accuracy (BLBP) sketching is not on the B200 path yet")
    _gpu_order_check(sketch.order)
    ranks, blocks, krylov = sketch.resolved_fixed_rank(sketch.order)
    return sketch, ranks, blocks, krylov


def gnhtsvt_randomized(a, transform=DEFAULT_TRANSFORM, penalty=None, tau: float = 0.0,
                       sketch: SketchConfig = None, sketch_override=None):
    """Singular-value thresholding accelerated by Tucker compression (GPU).

    ``a`` may be a numpy array (returned as numpy) or a torch tensor (returned
    as a CUDA tensor); float32 inputs stream in fp32, everything else in fp64.
    """
    if sketch is None:
        raise ValueError("a sketch configuration is required")
    if penalty is None:
        raise ValueError("a penalty is required")
    if tau < 0:
        raise ValueError("tau must be >= 0")
    transform = as_transform(transform)
    cm = a if isinstance(a, ColMajor) else to_device(a)
    dims = cm.dims
    if len(dims) < 3:
        raise ValueError(f"tensor order {len(dims)} < required 3")
    if any(n <= 0 for n in dims):
        raise ValueError(f"empty tensors are not supported, got shape {dims}")
    transform.check_shape(dims)
    sketch, ranks, blocks, krylov = _resolve(sketch, dims)
    out = empty_like(cm)
    _run_lrta(cm, out, ranks, blocks, krylov, sketch.seed, transform, penalty, tau,
              sketch_override)
    return out if isinstance(a, ColMajor) else from_device(out)


def _run_lrta(cm, out, ranks, blocks, krylov, seed, transform, penalty, tau, sketch_override=None,
              stream=None):
    lib = _lib.lib()
    dims = cm.dims
    d = _lib.i64(dims)
    rk, bl, kr = _lib.i64(ranks), _lib.i64(blocks), _lib.i64(krylov)
    nbytes = lib.tr_lrta_workspace(cm.dtype_code, len(dims), d, rk, bl, kr)
    if nbytes < 0:
        _lib.check(1)
    ws = workspace(nbytes)
    kind, p0, p1 = encode_penalty(penalty)
    tcode, tmats, talphas, keep_t = transform.device_args(dims)
    g0, g1, keep_g = _override_ptrs(sketch_override, cm)
    _lib.check(lib.tr_gnhtsvt_randomized(
        cm.dtype_code, ctypes.c_void_p(cm.ptr), ctypes.c_void_p(out.ptr), len(dims), d, rk, bl, kr,
        ctypes.c_uint64(int(seed) & (2 ** 64 - 1)), tcode, tmats, talphas, kind, p0, p1,
        float(tau), g0, g1, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
        _lib.stream_ptr(stream)))
    del keep_t, keep_g


def rsthosvd_bki(x, ranks, order=None, blocks=None, krylov=None, seed: int = 0,
                 strict_rank: bool = True, sketch_override=None):
    """Fixed-rank randomized Tucker compression of modes (0, 1) on the GPU.

    Factor columns carry the canonical sign (largest-|entry| positive).  With
    ``strict_rank`` a Krylov block that deflates below a target rank raises,
    like the reference.
    """
    import torch

    cm = x if isinstance(x, ColMajor) else to_device(x)
    dims = cm.dims
    order = (0, 1) if order is None else tuple(order)
    cfg = SketchConfig(mode="fixed-rank", order=order, ranks=tuple(ranks),
                       blocks=tuple(blocks) if blocks else None,
                       krylov=tuple(krylov) if krylov is not None else None, seed=seed)
    cfg.validate(dims)
    _gpu_order_check(order)
    rks, bls, krs = cfg.resolved_fixed_rank(order)
    lib = _lib.lib()
    d = _lib.i64(dims)
    rk, bl, kr = _lib.i64(rks), _lib.i64(bls), _lib.i64(krs)
    nbytes = lib.tr_lrta_workspace(cm.dtype_code, len(dims), d, rk, bl, kr)
    ws = workspace(nbytes)
    nf = int(math.prod(dims[2:]))
    f0 = torch.empty(dims[0] * rks[0], dtype=torch.float64, device="cuda")
    f1 = torch.empty(dims[1] * rks[1], dtype=torch.float64, device="cuda")
    core = torch.empty(rks[0] * rks[1] * nf, dtype=torch.float64, device="cuda")
    reff = torch.empty(2, dtype=torch.int64, device="cuda")
    g0, g1, keep = _override_ptrs(sketch_override, cm)
    _lib.check(lib.tr_rsthosvd_bki(
        cm.dtype_code, ctypes.c_void_p(cm.ptr), len(dims), d, rk, bl, kr,
        ctypes.c_uint64(int(seed) & (2 ** 64 - 1)), g0, g1, ctypes.c_void_p(f0.data_ptr()),
        ctypes.c_void_p(f1.data_ptr()), ctypes.c_void_p(core.data_ptr()),
        ctypes.c_void_p(reff.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
        _lib.stream_ptr()))
    del keep
    r0, r1 = (int(v) for v in reff.cpu())
    if strict_rank and (r0 < rks[0] or r1 < rks[1]):
        raise ValueError(f"Krylov block numerically rank deficient: ranks ({r0}, {r1}) < "
                         f"targets {tuple(rks)}")
    F0 = f0.reshape(rks[0], dims[0]).T[:, :r0]
    F1 = f1.reshape(rks[1], dims[1]).T[:, :r1]
    C = core.reshape(tuple(reversed((rks[0], rks[1]) + tuple(dims[2:])))).permute(
        *reversed(range(len(dims))))[:r0, :r1]
    factors = [F0, F1] + [None] * (len(dims) - 2)
    if cm.kind == "numpy":
        factors = [f.cpu().numpy() if f is not None else None for f in factors]
        C = C.cpu().numpy()
    return TuckerFactors(core=C, factors=factors, dims=tuple(dims))
