"""Parity of the native solvers with the oracle at BASELINE.json's own configs.

configs[0] (the CPU-runnable case): order-3 completion, 200x200x50 fp64, ground
truth = t-product of Gaussian factors 200x10x50 * 10x200x50 (tubal rank 10),
Frobenius-normalised, Bernoulli mask with 30% observed, randomized LRTA with
Krylov depth q = 2 and oversampling p = 5 (target rank 10 + 5 = 15, block
ceil(15 / 3) = 5), 100 ADMM iterations, seed 0.  Both completion solvers
(GNRHTC tenrec/solvers.py:287-289, GNHTC :292-295) run the full 100 sweeps on
the GPU and in the oracle (oracle/admm.py, fed the same Philox sketch stream);
L, E and every row of the residual / difference / multiplier histories must
agree to 1e-9 (fp64) and L to 1e-4 (fp32 twin).

configs[1] (the bench config): 1024x1024x128, exactly the bench's data
(bench.make_workload: rank-20 t-product + 10% outliers), 3 GNRHTC sweeps with
the bench's sketch (ranks 25, b = 7, q = 3).  The GPU f32 and fp64 runs are
compared with the fp64 oracle on the same input values: L and E after 3 sweeps
and each of the first sweep's three t-SVT outputs (G_k, one per gradient mode).

configs[3] shape (2048x2048x64 one-bit): the host sampling and the full GPU
solve run at the config's size; a 2-sweep oracle comparison pins the values.
"""

import numpy as np
import pytest

from oracle import admm, lrta, philox
from oracle.tensor_ops import TransformSpec

pytestmark = pytest.mark.gpu

MCP = (2, 2.5, 0.0)


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _tproduct_truth(n1, n2, n3, r, seed):
    """Gaussian factors n1 x r x n3 and r x n2 x n3, t-product along mode 3, ||X||_F = 1."""
    rng = np.random.default_rng(seed)
    a = np.fft.fft(rng.standard_normal((n1, r, n3)), axis=2)
    b = np.fft.fft(rng.standard_normal((r, n2, n3)), axis=2)
    x = np.real(np.fft.ifft(np.einsum("ikf,kjf->ijf", a, b), axis=2))
    return x / np.linalg.norm(x), rng


@pytest.fixture(scope="module")
def config0():
    x, rng = _tproduct_truth(200, 200, 50, 10, 0)
    mask = rng.random(x.shape) < 0.30
    return np.where(mask, x, 0.0), mask, x


def _oracle_threshold(ranks, blocks, krylov, seed, record=None):
    spec = TransformSpec("fft")

    def thr(a, tau):
        out = lrta.gnhtsvt_randomized(a, spec, MCP, tau, ranks, blocks, krylov, (0, 1),
                                      philox.PhiloxSketchSource(seed), canonical=True)
        if record is not None and len(record) < 3:
            record.append(out)
        return out

    return thr


C0_RANKS, C0_BLOCKS, C0_KRYLOV, C0_ITERS = (15, 15), (5, 5), (2, 2), 100


@pytest.fixture(scope="module")
def config0_oracle(config0):
    mobs, mask, _ = config0
    thr = _oracle_threshold(C0_RANKS, C0_BLOCKS, C0_KRYLOV, 0)
    lam = admm.default_lambda(mobs.shape)
    out = {}
    for noise_free in (False, True):
        out[noise_free] = admm.admm_complete(mobs, mask, thr, MCP, lam, (0, 1, 2),
                                             max_iters=C0_ITERS, tol=1e-30,
                                             noise_free=noise_free)
    return out


def _c0_cfg():
    import paper_2506_09594_b200 as pk

    sk = pk.SketchConfig(mode="fixed-rank", ranks=C0_RANKS, blocks=C0_BLOCKS, krylov=C0_KRYLOV,
                         seed=0)
    return pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                           max_iters=C0_ITERS, tol=1e-30)


@pytest.mark.parametrize("noise_free", [False, True], ids=["gnrhtc", "gnhtc"])
def test_config0_fp64_100_sweeps(cuda_lib, config0, config0_oracle, noise_free):
    import paper_2506_09594_b200 as pk

    mobs, mask, _ = config0
    lo, eo, hist = config0_oracle[noise_free]
    if noise_free:
        l, rep = pk.gnhtc(mobs, mask, _c0_cfg())
    else:
        l, e, rep = pk.gnrhtc(mobs, mask, _c0_cfg())
        assert _rel(e, eo) <= 1e-9
    assert rep.iterations == C0_ITERS
    assert _rel(l, lo) <= 1e-9, _rel(l, lo)
    # every history row: the Eq. (24) inf-norm residuals, the successive
    # Frobenius differences, the feasibility gaps, the multiplier norms and mu
    res = np.array(rep.residual_history)
    ores = np.array(hist["residuals"])
    scale = np.maximum(np.abs(ores), 1e-12 * np.abs(ores).max(axis=0, keepdims=True))
    assert np.max(np.abs(res - ores) / scale) <= 1e-7
    np.testing.assert_allclose(np.array(rep.diff_fro_history), np.array(hist["diff_fro"]),
                               rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(np.array(rep.feas_fro_history), np.array(hist["feas_fro"]),
                               rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(np.array(rep.multiplier_history), np.array(hist["multipliers"]),
                               rtol=1e-8)
    np.testing.assert_allclose(rep.mu_history, hist["mu"], rtol=1e-15)


@pytest.mark.parametrize("noise_free", [False, True], ids=["gnrhtc", "gnhtc"])
def test_config0_fp32_100_sweeps(cuda_lib, config0, config0_oracle, noise_free):
    import paper_2506_09594_b200 as pk

    mobs, mask, _ = config0
    lo, eo, _ = config0_oracle[noise_free]
    m32 = mobs.astype(np.float32)
    if noise_free:
        l, rep = pk.gnhtc(m32, mask, _c0_cfg())
    else:
        l, e, rep = pk.gnrhtc(m32, mask, _c0_cfg())
    assert l.dtype == np.float32 and rep.iterations == C0_ITERS
    assert _rel(l, lo) <= 1e-4, _rel(l, lo)


# -- configs[1]: the bench workload, 3 sweeps ----------------------------------

BENCH_SWEEPS = 3


@pytest.fixture(scope="module")
def bench_problem():
    import torch

    import bench

    flat = bench.make_workload(torch, bench.WORKLOAD["dims"], 1234)
    dims = bench.WORKLOAD["dims"]
    host = flat.reshape(tuple(reversed(dims))).permute(2, 1, 0).cpu().numpy()
    del flat
    torch.cuda.empty_cache()
    return np.asfortranarray(host)


@pytest.fixture(scope="module")
def bench_oracle(bench_problem):
    import bench

    w = bench.WORKLOAD
    x = bench_problem.astype(np.float64)
    rec = []
    thr = _oracle_threshold(w["ranks"], w["blocks"], w["krylov"], 7, rec)
    mask = np.ones(x.shape, dtype=bool)
    l, e, hist = admm.admm_complete(x, mask, thr, MCP, admm.default_lambda(x.shape), w["modes"],
                                    max_iters=BENCH_SWEEPS, tol=1e-30)
    return l, e, hist, rec


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_bench_config_sweeps_match_oracle(cuda_lib, bench_problem, bench_oracle, dtype):
    import torch

    import bench
    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200.solvers import NativeSolver
    from paper_2506_09594_b200.tensors import from_device, mask_to_device, to_device

    w = bench.WORKLOAD
    lo, eo, hist, g_oracle = bench_oracle
    x = bench_problem if dtype == "f32" else bench_problem.astype(np.float64)
    tol = 1e-4 if dtype == "f32" else 1e-9
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=w["ranks"], blocks=w["blocks"],
                         krylov=w["krylov"], seed=7)
    cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                          max_iters=BENCH_SWEEPS, tol=1e-30)
    cm = to_device(x)
    mask = mask_to_device(np.ones(x.shape, dtype=bool))
    run = NativeSolver("gnrhtc", cm, None, mask, cfg, w["modes"], cfg.lam_for(x.shape))
    try:
        res = []
        for it in range(BENCH_SWEEPS):
            res.append(run.step()[:5])
            if it == 0:
                # the first sweep's three t-SVT outputs (G_k of each gradient mode)
                for k in range(3):
                    gk = from_device(run.read(4 + k))
                    assert _rel(gk, g_oracle[k]) <= tol, (k, _rel(gk, g_oracle[k]))
                    del gk
        l = from_device(run.read(0))
        e = from_device(run.read(1))
    finally:
        run.close()
        torch.cuda.empty_cache()
    assert _rel(l, lo) <= tol, _rel(l, lo)
    assert _rel(e, eo) <= tol, _rel(e, eo)
    np.testing.assert_allclose(np.array(res), np.array(hist["residuals"]),
                               rtol=1e-3 if dtype == "f32" else 1e-7)


# -- configs[3] shape: one-bit at 2048 x 2048 x 64 ------------------------------

def test_onebit_config3_full_size(cuda_lib):
    """configs[3]: 2048x2048x64, tubal rank 10 scaled to max |x| = 1, one-bit
    observations on 50% of the entries, randomized LRTA (q = 2, p = 5),
    GNOBHTC.  The reference's observation model is a uniform dither of level
    theta plus optional Gaussian noise (tenrec/onebit.py:61-118); the config's
    noise of scale 0.1 is taken as sigma = 0.1 with theta = 1.5 (>= peak +
    3 sigma).  Two sweeps are compared with the oracle (fp64); the f32 stream
    (float32 aggregates J1, J2) runs the config's 30 iterations, checked for
    its box bound, finiteness and agreement with the fp64 run."""
    import torch

    import paper_2506_09594_b200 as pk

    dims = (2048, 2048, 64)
    x, _ = _tproduct_truth(*dims, 10, 3)
    x /= np.abs(x).max()
    obs = pk.onebit_observe(x, m=int(0.5 * x.size), theta=1.5, sigma=0.1, seed=11)
    del x
    sk = pk.SketchConfig(mode="fixed-rank", ranks=(15, 15), blocks=(5, 5), krylov=(2, 2), seed=0)

    def cfg(iters):
        return pk.SolverConfig.one_bit(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True,
                                       sketch=sk, max_iters=iters, tol=1e-30)

    lg, rep = pk.gnobhtc(obs, cfg(2), alpha=1.0)
    thr = _oracle_threshold((15, 15), (5, 5), (2, 2), 0)
    lam = admm.default_lambda(dims)
    lo, _, hist = admm.onebit_admm(obs.j1, obs.j2, float(obs.count), thr, lam, (0, 1, 2), 1.0,
                                   max_iters=2, tol=1e-30)
    assert _rel(lg, lo) <= 1e-9, _rel(lg, lo)
    np.testing.assert_allclose(np.array(rep.residual_history), np.array(hist["residuals"]),
                               rtol=1e-7, atol=1e-12)
    del lg, lo, hist
    l64, rep64 = pk.gnobhtc(obs, cfg(30), alpha=1.0)
    obs32 = pk.ObservationSet(dims=obs.dims, theta=obs.theta, indices=obs.indices,
                              signs=obs.signs, j1=obs.j1.astype(np.float32),
                              j2=obs.j2.astype(np.float32))
    l32, rep32 = pk.gnobhtc(obs32, cfg(30), alpha=1.0)
    assert l32.dtype == np.float32
    assert rep32.iterations == 30 and rep64.iterations == 30
    assert np.all(np.isfinite(l32)) and np.abs(l32).max() <= 1.0 + 1e-6
    assert _rel(l32, l64) <= 1e-4, _rel(l32, l64)
    torch.cuda.empty_cache()
