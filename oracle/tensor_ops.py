"""Column-major tensor algebra and trailing-mode transforms -- TEST INFRASTRUCTURE.

Restates tenrec/core.py (unfold/fold/mode product, norms) and
tenrec/transform.py (FFT / orthonormal DCT-II / explicit unitary-up-to-scale
transforms along modes >= 2, conjugate-mirror face pairing).  Every transform
is expressed here as a chain of mode products with a complex matrix, which is
exactly how the CUDA core-transform kernel applies it.
"""

from __future__ import annotations

import numpy as np

RESIDUE_RTOL = 1e-8  # tenrec/transform.py:37


class TransformError(ValueError):
    pass


def unfold(x, k):
    """Mode-k unfolding, earliest remaining mode fastest (tenrec/core.py:39-49)."""
    x = np.asarray(x)
    if not 0 <= k < x.ndim:
        raise ValueError("mode out of range")
    return np.moveaxis(x, k, 0).reshape((x.shape[k], -1), order="F")


def fold(m, k, dims):
    """Inverse of :func:`unfold` (tenrec/core.py:52-63)."""
    dims = tuple(int(v) for v in dims)
    rest = dims[:k] + dims[k + 1:]
    m = np.asarray(m)
    if m.shape != (dims[k], int(np.prod(rest, dtype=np.int64)) if rest else 1):
        raise ValueError("matrix does not match unfolding shape")
    return np.moveaxis(m.reshape((dims[k],) + rest, order="F"), 0, k)


def mode_product(x, u, k):
    """``x ×_k u`` (tenrec/core.py:66-78)."""
    dims = list(np.shape(x))
    dims[k] = u.shape[0]
    return fold(u @ unfold(x, k), k, dims)


def norms(x):
    """fro / l1 / tube1 / slice1 (tenrec/core.py:81-97)."""
    x = np.asarray(x)
    sq = np.abs(x) ** 2
    trailing = tuple(range(2, x.ndim))
    return {
        "fro": float(np.sqrt(sq.sum())),
        "l1": float(np.abs(x).sum()),
        "tube1": float(np.sqrt(sq.sum(axis=trailing)).sum()),
        "slice1": float(np.sqrt(sq.sum(axis=(0, 1))).sum()),
    }


# -- transforms as mode-product chains (tenrec/transform.py:44-183) ----------

def dft_matrix(n):
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n)


def dct2_ortho_matrix(n):
    """Orthonormal DCT-II, the matrix scipy's dctn(type=2, norm='ortho') applies."""
    k = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    c = np.cos(np.pi * (2 * j + 1) * k / (2 * n)) * np.sqrt(2.0 / n)
    c[0, :] *= 1.0 / np.sqrt(2.0)
    return c.astype(np.complex128)


class TransformSpec:
    """kind in {'fft', 'dct', 'explicit'}; explicit carries one matrix per trailing mode."""

    def __init__(self, kind="fft", matrices=None):
        self.kind = kind
        self.matrices = None
        self.alphas = None
        if kind == "explicit":
            mats = [np.asarray(m) for m in matrices]
            alphas = []
            for m in mats:
                if m.ndim != 2 or m.shape[0] != m.shape[1]:
                    raise TransformError("explicit transform matrices must be square")
                n = m.shape[0]
                gram = m @ m.conj().T
                a = float(np.real(np.trace(gram)) / n)
                if a <= 0 or np.max(np.abs(gram - a * np.eye(n))) > 1e-10 * max(1.0, a):
                    raise TransformError("matrix is not unitary up to scaling")
                alphas.append(a)
            self.matrices = mats
            self.alphas = alphas

    def mode_matrices(self, shape):
        """Forward matrices U_i and scalings alpha_i for every trailing mode."""
        trailing = tuple(shape[2:])
        if self.kind == "fft":
            return [dft_matrix(n) for n in trailing], [float(n) for n in trailing]
        if self.kind == "dct":
            return [dct2_ortho_matrix(n) for n in trailing], [1.0] * len(trailing)
        if len(trailing) != len(self.matrices) or any(
                m.shape[0] != n for m, n in zip(self.matrices, trailing)):
            raise TransformError("explicit transform does not match trailing modes")
        return [m.astype(np.complex128) for m in self.matrices], list(self.alphas)

    def rho(self, shape):
        _, alphas = self.mode_matrices(shape)
        return float(np.prod(alphas)) if alphas else 1.0

    def apply(self, x):
        x = np.asarray(x)
        if x.ndim < 3:
            raise TransformError("transforms require order >= 3")
        mats, _ = self.mode_matrices(x.shape)
        out = x.astype(np.complex128)
        for i, u in enumerate(mats):
            out = mode_product(out, u, 2 + i)
        return out

    def inverse(self, y, check_residue=True):
        y = np.asarray(y, dtype=np.complex128)
        mats, alphas = self.mode_matrices(y.shape)
        out = y
        for i in reversed(range(len(mats))):
            out = mode_product(out, mats[i].conj().T / alphas[i], 2 + i)
        real = out.real.copy()
        if check_residue:
            res = float(np.linalg.norm(out.imag))
            if res > RESIDUE_RTOL * max(float(np.linalg.norm(real)), 1e-300):
                raise TransformError("imaginary residue too large")
        return real

    def mirror_faces(self, shape):
        """FFT conjugate-symmetry partner of every flattened face (transform.py:169-183)."""
        if self.kind != "fft":
            return None
        trailing = tuple(shape[2:])
        nf = int(np.prod(trailing))
        idx = np.unravel_index(np.arange(nf), trailing, order="F")
        mir = tuple((n - t) % n for t, n in zip(idx, trailing))
        return np.ravel_multi_index(mir, trailing, order="F")


def as_faces(x):
    return np.reshape(x, (x.shape[0], x.shape[1], -1), order="F")


def from_faces(f, shape):
    return np.reshape(f, shape, order="F")


def canonical_faces(nf, mirror):
    if mirror is None:
        return np.arange(nf)
    return np.flatnonzero(np.arange(nf) <= mirror)


def face_singular_values(x, spec):
    """Singular values of every transformed face (transform.py:342-355)."""
    xf = as_faces(spec.apply(x))
    k = min(x.shape[0], x.shape[1])
    mirror = spec.mirror_faces(x.shape)
    out = np.zeros((k, xf.shape[2]))
    for j in canonical_faces(xf.shape[2], mirror):
        s = np.linalg.svd(xf[:, :, j], compute_uv=False)
        out[:, j] = s
        if mirror is not None and mirror[j] != j:
            out[:, int(mirror[j])] = s
    return out


def htnn(x, spec):
    """(1/rho) * sum of transformed-face singular values (transform.py:358-361)."""
    return float(face_singular_values(x, spec).sum() / spec.rho(x.shape))
