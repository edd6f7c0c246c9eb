"""Randomized low-rank tensor approximation and t-SVT -- TEST INFRASTRUCTURE.

Restates tenrec/sketch.py and tenrec/shrink.py:
  defl_qr            sketch.py:146-164   deflated pivoted QR (Algorithm 2)
  orthonormalize     sketch.py:167-185   Krylov basis: defl-QR at 1e-14*||K|| + re-QR
  sthosvd            sketch.py:188-208
  bki_factor         sketch.py:243-269   one mode of R-STHOSVD-BKI (Algorithm 1)
  rsthosvd_bki       sketch.py:211-270
  blbp_factor        sketch.py:287-352   one mode of AD-RSTHOSVD-BLBP (Algorithm 3)
  ad_rsthosvd_blbp   sketch.py:355-403
  gnhtsvt_randomized_blbp  sketch.py:406-456 with the fixed-accuracy compression
  gnhtt              shrink.py:57-73
  gnhtsvt            shrink.py:76-106
  gnhtsvt_randomized sketch.py:430-456

Two documented knobs make the oracle the checker for the GPU path:
  * ``source``: where sketch matrices come from.  ``NumpySketchSource``
    reproduces the reference's sequential PCG64 draws (pins the oracle to the
    reference); ``PhiloxSketchSource`` reproduces the GPU's counter-based
    draws (the GPU parity checker).
  * ``canonical``: the reference leaves the sign of every Ritz vector to
    LAPACK's ``eigh``.  The sign feeds the next mode's sketch, so the GPU path
    fixes it (largest-|entry| of each factor column made positive, first index
    on ties).  ``canonical=False`` reproduces the reference exactly.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from . import prox as P
from .tensor_ops import (as_faces, canonical_faces, fold, from_faces, mode_product,
                         unfold)


def defl_qr(a, tol):
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m == 0 or n == 0:
        return np.zeros((m, 0)), np.zeros((0, n)), 0
    q, r, piv = scipy.linalg.qr(a, mode="economic", pivoting=True)
    s = int(np.count_nonzero(np.abs(np.diag(r)) >= tol))
    r_out = np.empty((s, n))
    r_out[:, piv] = r[:s, :]
    return q[:, :s], r_out, s


def orthonormalize(k, rank_floor=0, strict=False):
    scale = np.linalg.norm(k)
    if scale == 0:
        raise ValueError("Krylov block is zero")
    q1, _, s = defl_qr(k, 1e-14 * scale)
    if strict and s < rank_floor:
        raise ValueError("Krylov block numerically rank deficient")
    q2, _ = np.linalg.qr(q1)
    return q2


def canonicalize_columns(f):
    """Flip each column so its largest-magnitude entry (first on ties) is positive."""
    f = np.array(f, copy=True)
    if f.size == 0:
        return f
    idx = np.argmax(np.abs(f), axis=0)
    sgn = np.sign(f[idx, np.arange(f.shape[1])])
    sgn[sgn == 0] = 1.0
    return f * sgn


def bki_factor(a, r, b, q, g, canonical=True):
    """Factor of one unfolding by block Krylov iteration (sketch.py:244-265).

    ``g`` is the (n, b) Gaussian sketch.  Returns an (m, r_eff) orthonormal
    factor; r_eff < r when the Krylov block deflates.
    """
    m, n = a.shape
    blk = a @ g
    pieces = []
    for i in range(q + 1):
        s = np.linalg.norm(blk)
        pieces.append(blk / s if s > 0 else blk)
        if i < q:  # the reference forms one more power it never uses
            blk = a @ (a.T @ pieces[-1])
    z = orthonormalize(np.hstack(pieces))
    r_eff = min(r, z.shape[1])
    w = a.T @ z
    _, vecs = np.linalg.eigh(w.T @ w)
    f = z @ vecs[:, z.shape[1] - r_eff:][:, ::-1]
    return canonicalize_columns(f) if canonical else f


def _defaults(ranks, blocks, krylov, n_modes):
    ranks = list(ranks)
    blocks = [max(1, int(np.ceil(r / 4))) for r in ranks] if blocks is None else list(blocks)
    krylov = [4] * n_modes if krylov is None else list(krylov)
    return ranks, blocks, krylov


def validate_fixed_rank(dims, order, ranks, blocks, krylov):
    """SketchConfig.validate for mode='fixed-rank' (sketch.py:83-105)."""
    for k in order:
        if not 0 <= k < len(dims):
            raise ValueError("processing order entry out of range")
    if not (len(ranks) == len(blocks) == len(krylov) == len(order)):
        raise ValueError("one entry per processed mode required")
    for k, r, b, qq in zip(order, ranks, blocks, krylov):
        if r > dims[k]:
            raise ValueError("rank exceeds mode length")
        if not 1 <= b <= r:
            raise ValueError("block size must satisfy 1 <= b <= r")
        if (qq + 1) * b < r:
            raise ValueError("(q+1)*b < rank")


def rsthosvd_bki(x, ranks, order=None, blocks=None, krylov=None, source=None,
                 canonical=True):
    """Returns (core, factors) like TuckerFactors (sketch.py:211-270)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.ndim
    order = tuple(range(d)) if order is None else tuple(order)
    ranks, blocks, krylov = _defaults(ranks, blocks, krylov, len(order))
    validate_fixed_rank(x.shape, order, ranks, blocks, krylov)
    factors = [None] * d
    core = x
    for step, (r, b, q, k) in enumerate(zip(ranks, blocks, krylov, order)):
        a = unfold(core, k)
        dims = list(core.shape)
        if np.linalg.norm(a) == 0.0:
            factors[k] = np.zeros((a.shape[0], 0))
            dims[k] = 0
            core = fold(np.zeros((0, a.shape[1])), k, dims)
            continue
        g = source.draw(step, a.shape[1], b)
        f = bki_factor(a, r, b, q, g, canonical)
        factors[k] = f
        dims[k] = f.shape[1]
        core = fold(f.T @ a, k, dims)
    return core, factors


def reconstruct(core, factors, dims):
    if any(n == 0 for n in core.shape):
        return np.zeros(dims)
    out = core
    for k, f in enumerate(factors):
        if f is not None:
            out = mode_product(out, f, k)
    return out


def sthosvd(x, ranks, order=None):
    x = np.asarray(x, dtype=np.float64)
    order = tuple(range(x.ndim)) if order is None else tuple(order)
    factors = [None] * x.ndim
    core = x
    for r, k in zip(ranks, order):
        a = unfold(core, k)
        u = np.linalg.svd(a, full_matrices=False)[0][:, :r]
        factors[k] = u
        dims = list(core.shape)
        dims[k] = r
        core = fold(u.T @ a, k, dims)
    return core, factors


# -- fixed accuracy: block Lanczos bidiagonalization (sketch.py:287-403) -----

def local_orthogonality_loss(blocks):
    blocks = [u for u in blocks if u.shape[1] > 0]
    loss = 0.0
    for i, u in enumerate(blocks):
        loss = max(loss, float(np.linalg.norm(u.T @ u - np.eye(u.shape[1]), 2)))
        if i:
            loss = max(loss, float(np.linalg.norm(blocks[i - 1].T @ u, 2)))
    return loss


def blbp_factor(a, eps, b, tol, draw, canonical=False):
    """One fixed-accuracy sweep; ``draw(n, cols)`` yields Gaussian blocks in order.

    ``canonical`` fixes the sign of every column of the finished factor
    (largest-|entry| positive), the convention of the GPU path: every step of
    the bidiagonalisation is equivariant under column sign flips of its
    blocks, so the factors then agree whatever sign convention each QR uses.
    """
    m, n = a.shape
    norm2 = float(np.linalg.norm(a) ** 2)
    if norm2 == 0.0:
        return np.zeros((m, 0)), [], 0.0, 0, 0
    v_cur, _ = np.linalg.qr(draw(n, min(b, n)))
    v_acc = v_cur
    blocks = []
    u_acc = np.zeros((m, 0))
    u_prev = l_prev = None
    energy, defl, it = norm2, 0, 0
    cap = 2 * int(np.ceil(min(m, n) / max(b, 1))) + 4
    while it < cap:
        it += 1
        w = a @ v_cur
        if u_prev is not None and u_prev.shape[1] > 0 and l_prev is not None:
            w = w - u_prev @ l_prev
        u_i, r_i, s_u = defl_qr(w, tol)
        keep = min(s_u, m - u_acc.shape[1])
        if keep < s_u:
            u_i, r_i, s_u = u_i[:, :keep], r_i[:keep, :], keep
        defl += w.shape[1] - s_u
        blocks.append(u_i)
        u_acc = np.hstack([u_acc, u_i])
        energy -= float(np.linalg.norm(r_i) ** 2)
        w2 = a.T @ u_i - v_cur @ r_i.T
        w2 = w2 - v_acc @ (v_acc.T @ w2)
        v_next, l_t, s_v = defl_qr(w2, tol)
        keep = min(s_v, n - v_acc.shape[1])
        if keep < s_v:
            v_next, l_t, s_v = v_next[:, :keep], l_t[:keep, :], keep
        v_acc = np.hstack([v_acc, v_next])
        l_next = l_t.T
        fill = min(b - s_v, n - v_acc.shape[1])
        if fill > 0:
            gn = draw(n, fill)
            gn = gn - v_acc @ (v_acc.T @ gn)
            vf, _ = np.linalg.qr(gn)
            v_acc = np.hstack([v_acc, vf])
            v_next = np.hstack([v_next, vf])
            l_next = np.hstack([l_next, np.zeros((s_u, vf.shape[1]))])
        energy -= float(np.linalg.norm(l_next) ** 2)
        if energy < eps ** 2 * norm2:
            break
        if s_u == 0 or v_next.shape[1] == 0 or u_acc.shape[1] >= m:
            break
        v_cur, u_prev, l_prev = v_next, u_i, l_next
    if canonical:
        u_acc = canonicalize_columns(u_acc)
    return u_acc, blocks, energy, defl, it


class PhiloxDraws:
    """The GPU path's Gaussian draws for block Lanczos: draw j of the call (a
    mode's start block or a fill block, counted across modes) is the (n, cols)
    Philox block of stream j (tenrec_b200.h: tr_tucker_create)."""

    def __init__(self, seed):
        from .philox import PhiloxSketchSource

        self.src = PhiloxSketchSource(seed)
        self.count = 0

    def __call__(self, n, cols):
        g = self.src.draw(self.count, n, cols)
        self.count += 1
        return g


def ad_rsthosvd_blbp(x, eps, block=10, defl_tol=None, order=None, rng=None, draw=None,
                     canonical=False):
    """sketch.py:355-403.  ``rng`` (numpy Generator, the reference's stream) or
    ``draw(n, cols)`` (e.g. PhiloxDraws) supplies the Gaussian blocks."""
    x = np.asarray(x, dtype=np.float64)
    order = tuple(range(x.ndim)) if order is None else tuple(order)
    if draw is None:
        rng = np.random.default_rng(0) if rng is None else rng
        draw = lambda n, c: rng.standard_normal((n, c))  # noqa: E731
    factors = [None] * x.ndim
    diag = {"energy": {}, "ranks": {}, "deflations": {}, "orth_loss": {}, "iterations": {}}
    core = x
    for k in order:
        a = unfold(core, k)
        nrm = float(np.linalg.norm(a))
        tol = defl_tol if defl_tol is not None else 1e-10 * max(nrm, 1e-300)
        f, blocks, energy, dfl, its = blbp_factor(a, eps, block, tol, draw, canonical)
        factors[k] = f
        diag["energy"][k] = energy
        diag["ranks"][k] = f.shape[1]
        diag["deflations"][k] = dfl
        diag["iterations"][k] = its
        diag["orth_loss"][k] = local_orthogonality_loss(blocks) if blocks else 0.0
        dims = list(core.shape)
        dims[k] = f.shape[1]
        core = fold(f.T @ a, k, dims)
    return core, factors, diag


# -- shrinkage ----------------------------------------------------------------

def gnhtt(a, pen, level, structure="entry"):
    """Entry / tube / slice group shrinkage (shrink.py:57-73, 49-54)."""
    a = np.asarray(a, dtype=np.float64)
    kind, p0, p1 = pen
    if level < 0:
        raise ValueError("shrinkage level must be >= 0")
    if structure == "entry":
        return P.prox(kind, p0, p1, level, a)
    if a.ndim < 3:
        raise ValueError("tube/slice shrinkage requires order >= 3")
    axes = tuple(range(2, a.ndim)) if structure == "tube" else (0, 1)
    gn = np.sqrt(np.sum(a ** 2, axis=axes, keepdims=True))
    sh = P.prox(kind, p0, p1, level, gn)
    with np.errstate(invalid="ignore", divide="ignore"):
        scale = np.where(gn > 0, sh / np.where(gn > 0, gn, 1.0), 0.0)
    return a * scale


def gnhtsvt(a, spec, pen, tau):
    """Transform-domain singular-value thresholding (shrink.py:76-106)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim < 3:
        raise ValueError("tensor order < 3")
    if tau < 0:
        raise ValueError("tau must be >= 0")
    kind, p0, p1 = pen
    af = as_faces(spec.apply(a))
    mirror = spec.mirror_faces(a.shape)
    out = np.empty_like(af)
    for j in canonical_faces(af.shape[2], mirror):
        face = af[:, :, j]
        if mirror is not None and mirror[j] == j:
            face = face.real
        u, s, vh = np.linalg.svd(face, full_matrices=False)
        rec = (u * P.prox(kind, p0, p1, tau, s)) @ vh
        out[:, :, j] = rec
        if mirror is not None and mirror[j] != j:
            out[:, :, int(mirror[j])] = np.conj(rec)
    return spec.inverse(from_faces(out, a.shape))


def gnhtsvt_randomized(a, spec, pen, tau, ranks, blocks=None, krylov=None, order=(0, 1),
                       source=None, canonical=True):
    """Tucker-compressed t-SVT (sketch.py:430-456), fixed-rank BKI compression."""
    a = np.asarray(a, dtype=np.float64)
    core, factors = rsthosvd_bki(a, ranks, order, blocks, krylov, source, canonical)
    if any(n == 0 for n in core.shape):
        return np.zeros(a.shape)
    return reconstruct(gnhtsvt(core, spec, pen, tau), factors, a.shape)


def gnhtsvt_randomized_blbp(a, spec, pen, tau, eps, block=10, defl_tol=None, order=(0, 1),
                            rng=None, draw=None, canonical=False):
    """Tucker-compressed t-SVT with fixed-accuracy BLBP compression (sketch.py:406-456)."""
    a = np.asarray(a, dtype=np.float64)
    core, factors, _ = ad_rsthosvd_blbp(a, eps, block, defl_tol, order, rng, draw, canonical)
    if any(n == 0 for n in core.shape):
        return np.zeros(a.shape)
    return reconstruct(gnhtsvt(core, spec, pen, tau), factors, a.shape)
