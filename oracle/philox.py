"""Counter-based Gaussian stream shared by the oracle and the CUDA sketch kernels.

TEST INFRASTRUCTURE (see ``oracle/__init__.py``).  The reference draws its
sketch matrices from ``numpy.random.default_rng(seed).standard_normal``
(tenrec/sketch.py:239,253), a sequential PCG64 stream that a GPU cannot
reproduce in parallel.  The B200 path instead draws every sketch entry from a
counter-based generator, so entry ``G[c, t]`` of the sketch used at processing
step ``p`` is a pure function of ``(seed, p, c*b + t)``.  This module is the
bit-for-bit CPU twin of ``gauss_at`` in ``paper_2506_09594_b200/csrc/philox.cuh``:

  * Philox4x32-10 (Salmon et al., SC'11): counter = (idx_lo, idx_hi,
    stream_lo, stream_hi), key = (seed_lo, seed_hi), ten rounds with the
    Weyl key bump between rounds.
  * two 53-bit uniforms from the four 32-bit words, Box-Muller to two
    normals; even flat indices take the cosine branch, odd the sine branch.

The flat index ``c*b + t`` is the row-major position inside an ``(n, b)``
matrix, the same order numpy fills ``standard_normal((n, b))``.  The GPU and
CPU agree to a few ulp (libm vs CUDA transcendental rounding); the parity
tolerances are orders of magnitude above that.
"""

from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)
_SH32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit words."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & _MASK32 for v in (c0, c1, c2, c3))
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _W0) & _MASK32
            k1 = (k1 + _W1) & _MASK32
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _SH32, p0 & _MASK32
        hi1, lo1 = p1 >> _SH32, p1 & _MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def gaussian_flat(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Standard normals at flat indices ``idx`` of stream ``stream``."""
    idx = np.asarray(idx, dtype=np.uint64)
    pair = idx >> np.uint64(1)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    stream = int(stream) & 0xFFFFFFFFFFFFFFFF
    x0, x1, x2, x3 = philox4x32_10(
        pair & _MASK32, pair >> _SH32,
        np.uint64(stream & 0xFFFFFFFF), np.uint64(stream >> 32),
        seed & 0xFFFFFFFF, seed >> 32,
    )
    two53 = 1.0 / 9007199254740992.0
    u1 = ((x0 >> np.uint64(5)).astype(np.float64) * 67108864.0
          + (x1 >> np.uint64(6)).astype(np.float64)) * two53
    u2 = ((x2 >> np.uint64(5)).astype(np.float64) * 67108864.0
          + (x3 >> np.uint64(6)).astype(np.float64)) * two53
    rad = np.sqrt(-2.0 * np.log(1.0 - u1))  # 1 - u1 in (0, 1]
    ang = 2.0 * np.pi * u2
    odd = (idx & np.uint64(1)).astype(bool)
    return np.where(odd, rad * np.sin(ang), rad * np.cos(ang))


def sketch_matrix(seed: int, stream: int, n: int, b: int) -> np.ndarray:
    """The ``(n, b)`` Gaussian sketch of processing step ``stream``."""
    flat = np.arange(int(n) * int(b), dtype=np.uint64)
    return gaussian_flat(seed, stream, flat).reshape(int(n), int(b))


class PhiloxSketchSource:
    """Sketch source for the oracle's BKI/BLBP: one stream per processing step.

    ``draw(step, n, b)`` returns the same matrix the CUDA kernels generate on
    the fly, so oracle and GPU consume identical sketches.
    """

    kind = "philox"

    def __init__(self, seed: int):
        self.seed = int(seed)

    def draw(self, step: int, n: int, b: int) -> np.ndarray:
        return sketch_matrix(self.seed, step, n, b)


class NumpySketchSource:
    """The reference's own sequential PCG64 stream (tenrec/sketch.py:239,253).

    Used only to pin the oracle against the reference bit-for-bit.
    """

    kind = "numpy"

    def __init__(self, seed: int):
        self.rng = np.random.default_rng(seed)

    def draw(self, step: int, n: int, b: int) -> np.ndarray:
        return self.rng.standard_normal((n, b))
