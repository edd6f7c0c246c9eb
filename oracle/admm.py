"""Circulant gradients, the FFT-diagonalised solve and the ADMM solvers -- TEST INFRASTRUCTURE.

Restates tenrec/gradient.py, tenrec/solvers.py and tenrec/onebit.py:
  grad / grad_adjoint        gradient.py:22-35
  solve_grad_system          gradient.py:90-106 (denominator gradient.py:63-80)
  kkt                        solvers.py:139-169
  admm_complete              solvers.py:204-284 (gnrhtc / gnhtc)
  data_fit_update            onebit.py:128-138
  onebit_admm                onebit.py:141-220 (gnobhtc / gnobrhtc)

The low-rank step is injected as ``threshold(a, tau)`` so the same loop runs
with the deterministic t-SVT or with the Tucker-randomized one.
"""

from __future__ import annotations

import numpy as np
import scipy.fft

from . import prox as P
from .lrta import gnhtt

RESIDUAL_NAMES = ("dL", "dE", "grad_gap", "dG", "fit_gap")
ONEBIT_RESIDUAL_NAMES = ("rel_dL", "box_gap", "grad_gap", "dG", "dL")


def grad(x, k):
    return np.roll(x, -1, axis=k) - x


def grad_adjoint(y, k):
    return np.roll(y, 1, axis=k) - y


def denominator(dims, modes):
    den = np.ones(dims)
    for k in modes:
        n = dims[k]
        shape = [1] * len(dims)
        shape[k] = n
        den = den + (4.0 * np.sin(np.pi * np.arange(n) / n) ** 2).reshape(shape)
    return den


def solve_grad_system(b, gmap, modes):
    """(I + sum_k D_k^T D_k) L = b + sum_k D_k^T g_k via the full d-dim FFT."""
    dims = b.shape
    num = scipy.fft.fftn(b)
    for k in modes:
        n = dims[k]
        shape = [1] * len(dims)
        shape[k] = n
        lam = (np.exp(2j * np.pi * np.arange(n) / n) - 1.0).reshape(shape)
        num += np.conj(lam) * scipy.fft.fftn(gmap[k])
    return np.real(scipy.fft.ifftn(num / denominator(dims, modes)))


def apply_operator(x, modes):
    out = np.array(x, dtype=np.float64, copy=True)
    for k in modes:
        out += grad_adjoint(grad(x, k), k)
    return out


def kkt(m, l, e, g, grad_l, l_prev, e_prev, g_prev):
    fit = m - l - e
    ks = list(g)
    inf = [float(np.max(np.abs(l - l_prev))), float(np.max(np.abs(e - e_prev))),
           max(float(np.max(np.abs(grad_l[k] - g[k]))) for k in ks),
           max(float(np.max(np.abs(g[k] - g_prev[k]))) for k in ks),
           float(np.max(np.abs(fit)))]
    fro = {"dL_fro": float(np.linalg.norm(l - l_prev)),
           "dE_fro": float(np.linalg.norm(e - e_prev)),
           "dG_fro": max(float(np.linalg.norm(g[k] - g_prev[k])) for k in ks),
           "fit_gap_fro": float(np.linalg.norm(fit)),
           "grad_gap_fro": max(float(np.linalg.norm(grad_l[k] - g[k])) for k in ks)}
    return inf, fro


def default_lambda(dims, xi=1.5):
    trailing = float(np.prod(dims[2:])) if len(dims) > 2 else 1.0
    return xi / float(np.sqrt(max(dims[0], dims[1]) * trailing))


def admm_complete(mobs, mask, threshold, psi, lam, modes, structure="entry", mu0=1e-3,
                  mu_max=1e10, growth=1.1, tol=1e-4, max_iters=500, noise_free=False,
                  pure_lowrank=False):
    """GNRHTC / GNHTC ADMM.  Returns (L, E, history dict)."""
    mobs = np.asarray(mobs, dtype=np.float64)
    maskf = np.asarray(mask, dtype=bool).astype(np.float64)
    dims = mobs.shape
    if pure_lowrank:
        modes = ("lowrank",)
        ap = lambda x, k: x  # noqa: E731
        solve = lambda b, gm: 0.5 * (b + gm["lowrank"])  # noqa: E731
    else:
        ap = grad
        solve = lambda b, gm: solve_grad_system(b, gm, modes)  # noqa: E731
    gamma = len(modes)
    l = np.zeros(dims)
    e = np.zeros(dims)
    g = {k: np.zeros(dims) for k in modes}
    lag = {k: np.zeros(dims) for k in modes}
    y = np.zeros(dims)
    mu = mu0
    hist = {"residuals": [], "diff_fro": [], "feas_fro": [], "multipliers": [], "mu": [],
            "iterations": 0, "converged": False}
    for _ in range(max_iters):
        b = mobs - e + y / mu
        l_new = solve(b, {k: g[k] - lag[k] / mu for k in modes})
        tau = 1.0 / (gamma * mu)
        grad_l = {k: ap(l_new, k) for k in modes}
        g_new = {k: threshold(grad_l[k] + lag[k] / mu, tau) for k in modes}
        h = mobs - l_new + y / mu
        if noise_free:
            e_new = (1.0 - maskf) * h
        else:
            e_new = maskf * gnhtt(maskf * h, psi, lam / mu, structure) + (1.0 - maskf) * h
        y = y + mu * (mobs - l_new - e_new)
        for k in modes:
            lag[k] = lag[k] + mu * (grad_l[k] - g_new[k])
        inf, fro = kkt(mobs, l_new, e_new, g_new, grad_l, l, e, g)
        hist["residuals"].append(inf)
        hist["diff_fro"].append([fro["dL_fro"], fro["dE_fro"], fro["dG_fro"]])
        hist["feas_fro"].append([fro["fit_gap_fro"], fro["grad_gap_fro"]])
        hist["multipliers"].append([float(np.linalg.norm(y)),
                                    max(float(np.linalg.norm(lag[k])) for k in modes)])
        hist["mu"].append(mu)
        l, e, g = l_new, e_new, g_new
        mu = min(mu_max, growth * mu)
        hist["iterations"] += 1
        if max(inf) <= tol and max(hist["diff_fro"][-1]) <= tol:
            hist["converged"] = True
            break
    return l, e, hist


# -- one-bit ------------------------------------------------------------------

def onebit_aggregates(dims, theta, indices, signs):
    n = int(np.prod(dims))
    j2 = np.bincount(indices, minlength=n).astype(np.float64).reshape(dims, order="F")
    j1 = (theta * np.bincount(indices, weights=signs.astype(np.float64), minlength=n)
          ).reshape(dims, order="F")
    return j1, j2


def data_fit_update(j1, j2, m, mu, z, y, alpha, s=None):
    num = j1 + m * mu * z - m * y
    if s is not None:
        num = num - j2 * s
    return np.clip(num / (j2 + m * mu), -alpha, alpha)


def onebit_admm(j1, j2, m, threshold, lam, modes, alpha, psi=None, lam2=None, robust=False,
                mu0=1e-6, mu_max=1e3, growth=1.05, tol=1e-4, max_iters=500):
    dims = j1.shape
    gamma = len(modes)
    observed = j2 > 0
    l = np.zeros(dims)
    s = np.zeros(dims)
    z = np.zeros(dims)
    g = {k: np.zeros(dims) for k in modes}
    lag = {k: np.zeros(dims) for k in modes}
    y = np.zeros(dims)
    mu = mu0
    hist = {"residuals": [], "multipliers": [], "mu": [], "iterations": 0, "converged": False}
    for it in range(max_iters):
        l_new = data_fit_update(j1, j2, m, mu, z, y, alpha, s=s if robust else None)
        if robust:
            s_new = np.zeros(dims)
            w = np.where(observed, j1 / np.maximum(j2, 1.0) - l_new, 0.0)
            for c in np.unique(j2[observed]):
                sel = j2 == c
                s_new[sel] = P.prox(psi[0], psi[1], psi[2], lam2 * m / float(c), w[sel])
            s = s_new
        z_new = solve_grad_system(l_new + y / mu, {k: g[k] - lag[k] / mu for k in modes}, modes)
        tau = lam / (gamma * mu)
        gz = {k: grad(z_new, k) for k in modes}
        g_new = {k: threshold(gz[k] + lag[k] / mu, tau) for k in modes}
        y = y + mu * (l_new - z_new)
        for k in modes:
            lag[k] = lag[k] + mu * (gz[k] - g_new[k])
        rel = float(np.linalg.norm(l_new - l)) / max(float(np.linalg.norm(l)), 1e-30)
        hist["residuals"].append([
            rel, float(np.max(np.abs(l_new - z_new))),
            max(float(np.max(np.abs(gz[k] - g_new[k]))) for k in modes),
            max(float(np.max(np.abs(g_new[k] - g[k]))) for k in modes),
            float(np.max(np.abs(l_new - l)))])
        hist["multipliers"].append([float(np.linalg.norm(y)),
                                    max(float(np.linalg.norm(lag[k])) for k in modes)])
        hist["mu"].append(mu)
        done = it > 0 and rel <= tol
        l, z, g = l_new, z_new, g_new
        mu = min(mu_max, growth * mu)
        hist["iterations"] += 1
        if done:
            hist["converged"] = True
            break
    return l, s, hist
