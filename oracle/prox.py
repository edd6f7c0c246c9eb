"""Scalar nonconvex penalties and proximity operators -- TEST INFRASTRUCTURE.

Restates tenrec/penalties.py.  A penalty is a ``(kind, p0, p1)`` triple, the
same encoding the C-ABI takes:

  kind  name        p0      p1      reference
  0     l1          -       -       penalties.py:67-75
  1     firm        gamma   -       penalties.py:104-116 (prox = MCP's)
  2     mcp         gamma   -       penalties.py:78-101
  3     scad        a       -       penalties.py:119-139
  4     lq          q       -       penalties.py:142-206
  5     capped-lq   q       theta   penalties.py:209-246
  6     log         gamma   -       penalties.py:249-270
"""

from __future__ import annotations

import numpy as np

KINDS = {"l1": 0, "firm": 1, "mcp": 2, "scad": 3, "lq": 4, "capped-lq": 5, "log": 6}
NEWTON_ITERS = 50     # penalties.py:154
NEWTON_TOL = 1e-12    # penalties.py:155
TIE = 1e-15           # penalties.py:243,270


def value(kind, p0, p1, t, mu):
    t = np.asarray(t, dtype=np.float64)
    if kind == 0:
        return mu * t
    if kind in (1, 2):
        g = p0
        return np.where(t <= g * mu, mu * t - t ** 2 / (2.0 * g), g * mu ** 2 / 2.0)
    if kind == 3:
        a = p0
        return np.where(t <= mu, mu * t,
                        np.where(t <= a * mu, (2.0 * a * mu * t - t ** 2 - mu ** 2) / (2.0 * (a - 1.0)),
                                 mu ** 2 * (a + 1.0) / 2.0))
    if kind == 4:
        return mu * t ** p0
    if kind == 5:
        return mu * np.minimum(t, p1) ** p0
    if kind == 6:
        return mu * np.log1p(t / p0)
    raise ValueError(kind)


def _lq_threshold(q, mu):
    if q == 1.0:
        return mu
    xh = (2.0 * mu * (1.0 - q)) ** (1.0 / (2.0 - q))
    return xh + mu * q * xh ** (q - 1.0)


def _lq_abs(q, mu, a):
    if q == 1.0:
        return np.maximum(a - mu, 0.0)
    out = np.zeros_like(a)
    live = a > _lq_threshold(q, mu)
    if not np.any(live):
        return out
    av = a[live]
    x = av.copy()
    converged = False
    for _ in range(NEWTON_ITERS):
        step = (x + mu * q * x ** (q - 1.0) - av) / (1.0 + mu * q * (q - 1.0) * x ** (q - 2.0))
        x = np.maximum(x - step, 1e-300)
        if np.max(np.abs(step)) < NEWTON_TOL:
            converged = True
            break
    if not converged:  # bisection on (xhat, a), penalties.py:196-206
        lo = np.full_like(av, (2.0 * mu * (1.0 - q)) ** (1.0 / (2.0 - q)))
        hi = av.copy()
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            neg = mid + mu * q * mid ** (q - 1.0) - av < 0
            lo = np.where(neg, mid, lo)
            hi = np.where(neg, hi, mid)
        x = 0.5 * (lo + hi)
    out[live] = x
    return out


def prox_abs(kind, p0, p1, mu, a):
    a = np.asarray(a, dtype=np.float64)
    if kind == 0:
        return np.maximum(a - mu, 0.0)
    if kind in (1, 2):
        g = p0
        return np.where(a <= mu, 0.0, np.where(a < g * mu, g * (a - mu) / (g - 1.0), a))
    if kind == 3:
        s = p0
        return np.where(a <= 2.0 * mu, np.maximum(a - mu, 0.0),
                        np.where(a <= s * mu, ((s - 1.0) * a - s * mu) / (s - 2.0), a))
    if kind == 4:
        return _lq_abs(p0, mu, a)
    if kind == 5:
        q, th = p0, p1
        inner = _lq_abs(q, mu, a)
        cands = [np.zeros_like(a), np.where(inner < th, inner, 0.0),
                 np.full_like(a, th), np.where(a > th, a, 0.0)]
        best = cands[0]
        fb = value(5, q, th, best, mu) + 0.5 * (best - a) ** 2
        for c in cands[1:]:
            f = value(5, q, th, c, mu) + 0.5 * (c - a) ** 2
            take = (f < fb - TIE) | ((np.abs(f - fb) <= TIE) & (c < best))
            best = np.where(take, c, best)
            fb = np.where(take, f, fb)
        return best
    if kind == 6:
        g = p0
        disc = (a + g) ** 2 - 4.0 * mu
        ok = disc >= 0
        root = np.where(ok, 0.5 * ((a - g) + np.sqrt(np.maximum(disc, 0.0))), 0.0)
        root = np.where(ok & (root > 0), root, 0.0)
        froot = value(6, g, 0.0, root, mu) + 0.5 * (root - a) ** 2
        return np.where(froot < 0.5 * a ** 2 - TIE, root, 0.0)
    raise ValueError(kind)


def prox(kind, p0, p1, mu, v):
    """Global minimiser of value(|x|, mu) + (x - v)^2 / 2 (penalties.py:45-61)."""
    v = np.asarray(v, dtype=np.float64)
    if mu < 0:
        raise ValueError("prox level mu must be >= 0")
    if mu == 0:
        return v.copy()
    return np.sign(v) * prox_abs(kind, p0, p1, float(mu), np.abs(v))


def from_reference(pen):
    """Map a reference/product penalty object to the (kind, p0, p1) triple."""
    name = type(pen).__name__
    table = {"L1": (0, 0.0, 0.0), "Firm": (1, getattr(pen, "gamma", 0.0), 0.0),
             "MCP": (2, getattr(pen, "gamma", 0.0), 0.0), "SCAD": (3, getattr(pen, "a", 0.0), 0.0),
             "Lq": (4, getattr(pen, "q", 0.0), 0.0),
             "CappedLq": (5, getattr(pen, "q", 0.0), getattr(pen, "theta", 0.0)),
             "LogPenalty": (6, getattr(pen, "gamma", 0.0), 0.0)}
    kind, p0, p1 = table[name]
    return kind, float(p0), float(p1)
