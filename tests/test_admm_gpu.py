"""Parity of the native ADMM solvers with the reference (golden runs) and the oracle.

Deterministic-threshold runs (small faces) are compared directly with the
reference's own outputs and residual histories recorded in
tests/golden/reference_vectors.npz; randomized runs against the oracle fed the
same Philox sketch stream.
"""

import numpy as np
import pytest

from oracle import admm, lrta, philox
from oracle.tensor_ops import TransformSpec

pytestmark = pytest.mark.gpu


def _cfg(tag, **kw):
    import paper_2506_09594_b200 as pk
    base = dict(max_iters=15)
    if tag == "tube":
        base.update(structure="tube", psi=pk.L1())
    if tag == "pure":
        base.update(pure_lowrank=True)
    base.update(kw)
    return pk.SolverConfig(**base)


@pytest.mark.parametrize("tag", ["det", "tube", "pure"])
def test_gnrhtc_matches_reference(cuda_lib, golden, tag):
    import paper_2506_09594_b200 as pk
    mobs, mask = golden["admm_mobs"], golden["admm_mask"]
    l, e, rep = pk.gnrhtc(mobs, mask, _cfg(tag))
    np.testing.assert_allclose(l, golden[f"admm_{tag}_l"], atol=1e-9)
    np.testing.assert_allclose(e, golden[f"admm_{tag}_e"], atol=1e-9)
    np.testing.assert_allclose(np.array(rep.residual_history), golden[f"admm_{tag}_res"],
                               rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(np.array(rep.diff_fro_history), golden[f"admm_{tag}_dfro"],
                               rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(np.array(rep.multiplier_history), golden[f"admm_{tag}_mult"],
                               rtol=1e-8)
    assert rep.iterations == 15 and len(rep.mu_history) == 15


def test_gnhtc_matches_reference(cuda_lib, golden):
    import paper_2506_09594_b200 as pk
    l, rep = pk.gnhtc(golden["admm_mobs"], golden["admm_mask"], _cfg("nf"))
    np.testing.assert_allclose(l, golden["admm_nf_l"], atol=1e-9)
    np.testing.assert_allclose(np.array(rep.residual_history), golden["admm_nf_res"], rtol=1e-6,
                               atol=1e-9)


def _oracle_rnd(mobs, mask, iters, ranks, blocks, krylov, seed):
    spec = TransformSpec("fft")
    mcp = (2, 2.5, 0.0)

    def thr(a, tau):
        return lrta.gnhtsvt_randomized(a, spec, mcp, tau, ranks, blocks, krylov, (0, 1),
                                       philox.PhiloxSketchSource(seed), canonical=True)

    return admm.admm_complete(mobs, mask, thr, mcp, admm.default_lambda(mobs.shape), (0, 1, 2),
                              max_iters=iters)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_randomized_gnrhtc_matches_oracle(cuda_lib, golden, dtype):
    import paper_2506_09594_b200 as pk
    mobs, mask = golden["admm_mobs"], golden["admm_mask"]
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(6, 5), blocks=(2, 2),
                         krylov=(2, 2), seed=3)
    cfg = pk.SolverConfig(max_iters=10, randomized=True, sketch=sk)
    xin = mobs if dtype == "f64" else mobs.astype(np.float32)
    l, e, rep = pk.gnrhtc(xin, mask, cfg)
    lo, eo, hist = _oracle_rnd(mobs, mask, 10, (6, 5), (2, 2), (2, 2), 3)
    rel = np.linalg.norm(l - lo) / np.linalg.norm(lo)
    assert rel <= (1e-9 if dtype == "f64" else 1e-4), rel
    np.testing.assert_allclose(np.array(rep.residual_history), np.array(hist["residuals"]),
                               rtol=1e-6 if dtype == "f64" else 5e-3, atol=1e-7)


def _lowrank_problem(seed=5):
    from oracle.tensor_ops import mode_product
    rng = np.random.default_rng(seed)
    core = rng.standard_normal((4, 4, 16))
    x = mode_product(mode_product(core, rng.standard_normal((64, 4)), 0),
                     rng.standard_normal((64, 4)), 1)
    mask = rng.random(x.shape) < 0.7
    return np.where(mask, x, 0.0), mask


@pytest.mark.parametrize("ranks", [(4, 4), (8, 8)])
def test_larger_randomized_power_of_two(cuda_lib, ranks):
    """64 x 64 x 16: radix-2 FFT passes, fused panels, tcgen05 projection.

    ranks (4, 4) = the signal's multilinear rank; ranks (8, 8) makes Ritz
    vectors 5-8 span a near-null space.  Both meet the 1e-4 fp32 bar after 6
    sweeps (tools/f32_drift_probe.py: 2.2e-5 and 3.4e-5 on the B200; the
    CUDA-core fallback panels, TR_NO_PANEL, drift to 4.5e-4 on (8, 8)).
    """
    fp32_tol = 1e-4
    import paper_2506_09594_b200 as pk
    mobs, mask = _lowrank_problem()
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=ranks, blocks=(2, 2),
                         krylov=(3, 3), seed=1)
    cfg = pk.SolverConfig(max_iters=6, randomized=True, sketch=sk)
    l, e, rep = pk.gnrhtc(mobs, mask, cfg)
    lo, eo, hist = _oracle_rnd(mobs, mask, 6, ranks, (2, 2), (3, 3), 1)
    assert np.linalg.norm(l - lo) / np.linalg.norm(lo) <= 1e-9
    l32, _, rep32 = pk.gnrhtc(mobs.astype(np.float32), mask, cfg)
    assert np.linalg.norm(l32 - lo) / np.linalg.norm(lo) <= fp32_tol


def test_onebit_matches_reference(cuda_lib, golden):
    import paper_2506_09594_b200 as pk
    obs = pk.ObservationSet(dims=golden["ob_j1"].shape, theta=float(golden["ob_theta"]),
                            indices=golden["ob_idx"], signs=golden["ob_sgn"])
    np.testing.assert_array_equal(obs.j1, golden["ob_j1"])
    l, rep = pk.gnobhtc(obs, pk.SolverConfig.one_bit(max_iters=12))
    np.testing.assert_allclose(l, golden["ob_l"], atol=1e-9)
    np.testing.assert_allclose(np.array(rep.residual_history), golden["ob_res"], rtol=1e-6,
                               atol=1e-9)
    l, s, rep = pk.gnobrhtc(obs, pk.SolverConfig.one_bit(max_iters=12, lam2=0.05, psi=pk.L1()))
    np.testing.assert_allclose(l, golden["obr_l"], atol=1e-9)
    np.testing.assert_allclose(s, golden["obr_s"], atol=1e-9)
    np.testing.assert_allclose(np.array(rep.residual_history), golden["obr_res"], rtol=1e-6,
                               atol=1e-9)


def test_solver_input_errors(cuda_lib, golden):
    import paper_2506_09594_b200 as pk
    mobs, mask = golden["admm_mobs"], golden["admm_mask"]
    with pytest.raises(ValueError, match="empty"):
        pk.gnrhtc(mobs * 0, np.zeros_like(mask), pk.SolverConfig(max_iters=1))
    bad = mobs.copy()
    bad[~mask] = 1.0
    with pytest.raises(ValueError, match="zero outside"):
        pk.gnrhtc(bad, mask, pk.SolverConfig(max_iters=1))
    with pytest.raises(ValueError, match="sketch"):
        pk.gnrhtc(mobs, mask, pk.SolverConfig(randomized=True))


def test_zero_problem_converges_immediately(cuda_lib):
    import paper_2506_09594_b200 as pk
    mask = np.ones((6, 5, 4), dtype=bool)
    l, e, rep = pk.gnrhtc(np.zeros((6, 5, 4)), mask, pk.SolverConfig(max_iters=5))
    assert rep.converged and rep.iterations == 1
    assert not l.any() and not e.any()


def test_deterministic_large_faces_match_oracle(cuda_lib):
    """Deterministic GNRHTC (the reference's default, randomized=False) with
    face slices larger than 64 x 64: the face SVT keeps its working copy and
    rotations in global scratch (k_face_svt_g).  96 x 80 x 6, 4 sweeps, fp64."""
    import paper_2506_09594_b200 as pk
    from oracle.tensor_ops import mode_product
    rng = np.random.default_rng(9)
    core = rng.standard_normal((5, 5, 6))
    x = mode_product(mode_product(core, rng.standard_normal((96, 5)), 0),
                     rng.standard_normal((80, 5)), 1)
    mask = rng.random(x.shape) < 0.6
    mobs = np.where(mask, x, 0.0)
    l, e, rep = pk.gnrhtc(mobs, mask, pk.SolverConfig(max_iters=4))
    spec = TransformSpec("fft")
    mcp = (2, 2.5, 0.0)
    lo, eo, hist = admm.admm_complete(mobs, mask, lambda a, tau: lrta.gnhtsvt(a, spec, mcp, tau),
                                      mcp, admm.default_lambda(mobs.shape), (0, 1, 2),
                                      max_iters=4)
    assert np.linalg.norm(l - lo) / np.linalg.norm(lo) <= 1e-9
    assert np.linalg.norm(e - eo) / max(np.linalg.norm(eo), 1e-300) <= 1e-9
    np.testing.assert_allclose(np.array(rep.residual_history), np.array(hist["residuals"]),
                               rtol=1e-6, atol=1e-9)
    # the fp32 stream through the same large-face path
    l32, e32, _ = pk.gnrhtc(mobs.astype(np.float32), mask, pk.SolverConfig(max_iters=4))
    assert np.linalg.norm(l32 - lo) / np.linalg.norm(lo) <= 1e-4


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lookahead_is_bit_identical(cuda_lib, dtype):
    """tr_admm_lookahead only moves the next sweep's L-solve ahead of the host's
    read-back: residual histories, L and E must not change by a bit, whether the
    loop runs to max_iters or stops early with a lookahead in flight."""
    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200.solvers import NativeSolver
    from paper_2506_09594_b200.tensors import from_device, mask_to_device, to_device

    rng = np.random.default_rng(3)
    x = rng.standard_normal((32, 16, 3)) @ rng.standard_normal((3, 24))
    x = np.moveaxis(x, 1, 2).astype(dtype)  # 32 x 24 x 16, low rank along mode 1
    x = np.asfortranarray(x + 0.01 * rng.standard_normal(x.shape).astype(dtype))
    mask = rng.random(x.shape) < 0.6
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(6, 6), blocks=(3, 3),
                         krylov=(2, 2), seed=11)
    cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk, tol=1e-30)

    def run(lookahead, sweeps):
        cm = to_device(x * mask)
        s = NativeSolver("gnrhtc", cm, None, mask_to_device(mask), cfg, cfg.device_modes(x.shape),
                         cfg.lam_for(x.shape))
        hist = [s.step(last=not lookahead) for _ in range(sweeps)]
        out = from_device(s.read(0)).copy(), from_device(s.read(1)).copy()
        s.close()
        return np.array(hist), out

    h0, (l0, e0) = run(False, 7)
    h1, (l1, e1) = run(True, 7)   # stops with the 8th sweep's L-solve enqueued
    assert np.array_equal(h0, h1)
    assert np.array_equal(l0, l1) and np.array_equal(e0, e1)
