"""Randomized Tucker sketching and the randomized t-SVT on the B200.

Drop-in for tenrec/sketch.py:
  SketchConfig          sketch.py:64-126 (same fields, defaults and errors)
  TuckerFactors         sketch.py:39-61
  BLBPDiagnostics       sketch.py:129-143
  rsthosvd_bki          sketch.py:211-270  -> C ABI tr_rsthosvd_bki (order (0, 1))
                                              or the generic engine tr_tucker_*
  ad_rsthosvd_blbp      sketch.py:355-403  -> tr_tucker_* (block Lanczos)
  gnhtsvt_randomized    sketch.py:430-456  -> tr_gnhtsvt_randomized (fixed-rank,
                                              order (0, 1): the ADMM hot path)
                                              or tr_tucker_create + tr_tucker_svt

Sketch matrices come from the counter-based Philox stream (entry (c, t) of
processing step p is N(0,1) at (seed, p, c*b + t)), so results are
deterministic per seed and identical to the oracle fed the same stream.
``sketch_override=(g0, g1)`` replays externally drawn matrices instead.  The
block Lanczos path numbers its Gaussian draws in call order across all modes:
draw j (the start block of a mode or a fill block) is the (n, cols) matrix of
entries N(0,1) at (seed, j, c*cols + t).
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


@dataclass
class BLBPDiagnostics:
    """Per-mode traces of the fixed-accuracy sweep (sketch.py:129-143)."""

    energy_estimates: dict = field(default_factory=dict)
    ranks: dict = field(default_factory=dict)
    deflations: dict = field(default_factory=dict)
    orth_loss: dict = field(default_factory=dict)
    iterations: dict = field(default_factory=dict)

    @property
    def implied_error(self) -> float:
        total = sum(max(e, 0.0) for e in self.energy_estimates.values())
        return float(np.sqrt(total))


class TuckerRun:
    """One compression by the generic device engine (C ABI tr_tucker_*):
    factors, core and diagnostics stay on the device until read."""

    def __init__(self, cm: ColMajor, sketch: SketchConfig, order, stream=None):
        self.lib = _lib.lib()
        self.cm = cm
        self.dims = cm.dims
        d = len(self.dims)
        order = tuple(int(k) for k in order)
        if sketch.mode == "fixed-rank":
            ranks, blocks, krylov = sketch.resolved_fixed_rank(order)
            mode = 0
        else:
            ranks = blocks = krylov = [0] * len(order)
            mode = 1
        handle = ctypes.c_void_p()
        _lib.check(self.lib.tr_tucker_create(
            cm.dtype_code, ctypes.c_void_p(cm.ptr), d, _lib.i64(self.dims), mode, len(order),
            _lib.i64(order), _lib.i64(ranks), _lib.i64(blocks), _lib.i64(krylov),
            float(sketch.eps), int(sketch.block),
            float(sketch.defl_tol) if sketch.defl_tol is not None else 0.0,
            ctypes.c_uint64(int(sketch.seed) & (2 ** 64 - 1)), _lib.stream_ptr(stream),
            ctypes.byref(handle)))
        self.handle = handle
        cdims = (ctypes.c_int64 * d)()
        rks = (ctypes.c_int64 * d)()
        proc = (ctypes.c_int64 * d)()
        en = (ctypes.c_double * d)()
        dfl = (ctypes.c_int64 * d)()
        its = (ctypes.c_int64 * d)()
        orl = (ctypes.c_double * d)()
        _lib.check(self.lib.tr_tucker_info(handle, cdims, rks, proc, en, dfl, its, orl))
        self.core_dims = tuple(int(v) for v in cdims)
        self.ranks = tuple(int(v) for v in rks)
        self.processed = tuple(bool(v) for v in proc)
        self.order = order
        self.diag = BLBPDiagnostics()
        for k in order:
            self.diag.energy_estimates[k] = float(en[k])
            self.diag.ranks[k] = int(rks[k])
            self.diag.deflations[k] = int(dfl[k])
            self.diag.iterations[k] = int(its[k])
            self.diag.orth_loss[k] = float(orl[k])

    def factors(self):
        import torch

        out = []
        for k, n in enumerate(self.dims):
            if not self.processed[k]:
                out.append(None)
                continue
            r = self.ranks[k]
            f = torch.empty(max(n * r, 1), dtype=torch.float64, device="cuda")
            if r:
                _lib.check(self.lib.tr_tucker_read(self.handle, k, ctypes.c_void_p(f.data_ptr()),
                                                   _lib.stream_ptr()))
            out.append(f[:n * r].reshape(r, n).T)
        return out

    def core(self):
        import torch

        nc = int(math.prod(self.core_dims))
        c = torch.empty(max(nc, 1), dtype=torch.float64, device="cuda")
        if nc:
            _lib.check(self.lib.tr_tucker_read(self.handle, -1, ctypes.c_void_p(c.data_ptr()),
                                               _lib.stream_ptr()))
        d = len(self.core_dims)
        return c[:nc].reshape(tuple(reversed(self.core_dims))).permute(*reversed(range(d)))

    def svt(self, transform, penalty, tau, out: ColMajor, stream=None):
        kind, p0, p1 = encode_penalty(penalty)
        tcode, tmats, talphas, keep = transform.device_args(self.core_dims) \
            if transform.kind == "explicit" else transform.device_args(self.dims)
        _lib.check(self.lib.tr_tucker_svt(self.handle, tcode, tmats, talphas, kind, p0, p1,
                                          float(tau), ctypes.c_void_p(out.ptr),
                                          _lib.stream_ptr(stream)))
        del keep

    def tucker_factors(self, as_numpy: bool):
        factors = self.factors()
        core = self.core()
        if as_numpy:
            factors = [f.cpu().numpy() if f is not None else None for f in factors]
            core = core.cpu().numpy()
        return TuckerFactors(core=core, factors=factors, dims=tuple(self.dims))

    def close(self):
        if self.handle:
            self.lib.tr_tucker_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _fast_path(sketch: SketchConfig, order) -> bool:
    """The asynchronous fused launch sequence (lrta.cu) handles fixed-rank
    compression of modes (0, 1) -- the ADMM hot path; the generic engine the rest."""
    return sketch.mode == "fixed-rank" and tuple(order) == (0, 1)


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


def _with_default_order(sketch: SketchConfig) -> SketchConfig:
    """gnhtsvt_randomized's default: compress modes 0 and 1 only (sketch.py:444-451)."""
    if sketch.order is not None:
        return sketch
    return SketchConfig(mode=sketch.mode, order=(0, 1), ranks=sketch.ranks,
                        blocks=sketch.blocks, krylov=sketch.krylov, eps=sketch.eps,
                        block=sketch.block, defl_tol=sketch.defl_tol, seed=sketch.seed)


def _resolve(sketch: SketchConfig, dims):
    """(sketch, ranks, blocks, krylov) of the fused fixed-rank (0, 1) path."""
    sketch = _with_default_order(sketch)
    sketch.validate(dims)
    if not _fast_path(sketch, sketch.order):
        raise ValueError("the fused path compresses modes (0, 1) with a fixed-rank sketch")
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
    sketch = _with_default_order(sketch)
    sketch.validate(dims)
    out = empty_like(cm)
    if _fast_path(sketch, sketch.order):
        transform.check_shape(dims)
        ranks, blocks, krylov = sketch.resolved_fixed_rank(sketch.order)
        _run_lrta(cm, out, ranks, blocks, krylov, sketch.seed, transform, penalty, tau,
                  sketch_override)
    else:
        if sketch_override is not None:
            raise ValueError("sketch_override applies to the fixed-rank (0, 1) path only")
        run = TuckerRun(cm, sketch, sketch.order)
        try:
            if transform.kind == "explicit":
                transform.check_shape(run.core_dims)
            run.svt(transform, penalty, tau, out)
        finally:
            run.close()
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
    """Fixed-rank randomized Tucker compression on the GPU (sketch.py:211-270).

    ``order`` defaults to every mode, like the reference.  Factor columns
    carry the canonical sign (largest-|entry| positive).  With ``strict_rank``
    a Krylov block that deflates below a target rank raises, like the
    reference; an all-zero input gives a rank-0 structure.
    """
    import torch

    cm = x if isinstance(x, ColMajor) else to_device(x)
    dims = cm.dims
    order = tuple(range(len(dims))) if order is None else tuple(int(k) for k in order)
    cfg = SketchConfig(mode="fixed-rank", order=order, ranks=tuple(ranks),
                       blocks=tuple(blocks) if blocks else None,
                       krylov=tuple(krylov) if krylov is not None else None, seed=seed)
    cfg.validate(dims)
    rks, bls, krs = cfg.resolved_fixed_rank(order)
    if order != (0, 1) or len(dims) < 3 or not bool(cm.flat.any()):
        if sketch_override is not None:
            raise ValueError("sketch_override applies to the order (0, 1) path only")
        run = TuckerRun(cm, cfg, order)
        try:
            for k, r in zip(order, rks):
                if run.ranks[k] == 0:
                    break  # a zero unfolding: rank-0 structure, no rank check (sketch.py:246-252)
                if strict_rank and run.ranks[k] < r:
                    raise ValueError(f"Krylov block numerically rank deficient on mode {k}: "
                                     f"rank {run.ranks[k]} < target {r}")
            return run.tucker_factors(cm.kind == "numpy")
        finally:
            run.close()
    lib = _lib.lib()
    d = _lib.i64(dims)
    rk, bl, kr = _lib.i64(rks), _lib.i64(bls), _lib.i64(krs)
    nbytes = lib.tr_lrta_workspace(cm.dtype_code, len(dims), d, rk, bl, kr)
    if nbytes < 0:
        _lib.check(1)
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


def ad_rsthosvd_blbp(x, eps: float, block: int = 10, defl_tol: float = None, order=None,
                     seed: int = 0):
    """Fixed-accuracy Tucker compression by block Lanczos bidiagonalisation
    (sketch.py:355-403) on the GPU.  Returns ``(TuckerFactors, BLBPDiagnostics)``."""
    cm = x if isinstance(x, ColMajor) else to_device(x)
    dims = cm.dims
    order = tuple(range(len(dims))) if order is None else tuple(int(k) for k in order)
    cfg = SketchConfig(mode="fixed-accuracy", order=order, eps=eps, block=block,
                       defl_tol=defl_tol, seed=seed)
    cfg.validate(dims)
    if defl_tol is not None:
        # sketch.py:384-388 (checked against ||x||_F, which bounds every mode's core)
        import warnings

        nrm = float(cm.flat.double().norm())
        if nrm > 0 and defl_tol >= nrm:
            warnings.warn(f"deflation tolerance {defl_tol:.3e} >= unfolding norm {nrm:.3e} "
                          f"on mode {order[0]}", stacklevel=2)
    run = TuckerRun(cm, cfg, order)
    try:
        return run.tucker_factors(cm.kind == "numpy"), run.diag
    finally:
        run.close()
