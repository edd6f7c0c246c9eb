"""The generic Tucker engine on the GPU (tr_tucker_*): fixed-accuracy block
Lanczos bidiagonalisation (tenrec/sketch.py:287-403), fixed-rank compression in
any processing order (sketch.py:211-270) and the Tucker-compressed t-SVT on
top of either (sketch.py:406-456), against the oracle fed the same Philox
draws with the canonical column signs.  The oracle itself is pinned to the
reference's own outputs on the same inputs (tests/test_oracle_golden.py).
"""

import numpy as np
import pytest

from oracle import lrta, philox
from oracle.tensor_ops import TransformSpec

pytestmark = pytest.mark.gpu

MCP = (2, 2.5, 0.0)


def _rel(a, b):
    b = np.asarray(b)
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _blbp_args(golden, i):
    pre = f"blbp{i}_"
    dt = float(golden[pre + "defl_tol"])
    return (golden[pre + "in"], float(golden[pre + "eps"]), int(golden[pre + "block"]),
            None if dt < 0 else dt, tuple(int(k) for k in golden[pre + "order"]),
            int(golden[pre + "seed"]))


@pytest.mark.parametrize("i", range(5))
def test_blbp_golden_inputs_match_oracle(cuda_lib, golden, i):
    import paper_2506_09594_b200 as pk

    a, eps, block, dtol, order, seed = _blbp_args(golden, i)
    tf, diag = pk.ad_rsthosvd_blbp(a, eps, block=block, defl_tol=dtol, order=order, seed=seed)
    core, factors, od = lrta.ad_rsthosvd_blbp(a, eps, block, dtol, order,
                                              draw=lrta.PhiloxDraws(seed), canonical=True)
    for k in order:
        assert tf.factors[k].shape == factors[k].shape, (k, tf.factors[k].shape, factors[k].shape)
        assert _rel(tf.factors[k], factors[k]) <= 1e-9, (k, _rel(tf.factors[k], factors[k]))
        assert diag.ranks[k] == od["ranks"][k]
        assert diag.iterations[k] == od["iterations"][k]
        assert diag.deflations[k] == od["deflations"][k]
        assert abs(diag.energy_estimates[k] - od["energy"][k]) <= 1e-9 * float(np.sum(a * a))
        assert abs(diag.orth_loss[k] - od["orth_loss"][k]) <= 1e-9
    assert tf.core.shape == core.shape
    assert _rel(tf.core, core) <= 1e-9
    if a.ndim >= 3:
        sk = pk.SketchConfig(mode="fixed-accuracy", order=order, eps=eps, block=block,
                             defl_tol=dtol, seed=seed)
        got = pk.gnhtsvt_randomized(a, pk.Transform.fft(), pk.MCP(2.5), 0.3, sk)
        ref = lrta.gnhtsvt_randomized_blbp(a, TransformSpec("fft"), MCP, 0.3, eps, block, dtol,
                                           order, draw=lrta.PhiloxDraws(seed), canonical=True)
        assert _rel(got, ref) <= 1e-9, _rel(got, ref)
        # fp32 stream: the block Lanczos passes accumulate in fp64 (their
        # deflation test runs at 1e-10 ||A||), so the fp32 run reproduces the
        # oracle on the same fp32 input values
        a32 = a.astype(np.float32)
        got32 = pk.gnhtsvt_randomized(a32, pk.Transform.fft(), pk.MCP(2.5), 0.3, sk)
        ref32 = lrta.gnhtsvt_randomized_blbp(a32.astype(np.float64), TransformSpec("fft"), MCP,
                                             0.3, eps, block, dtol, order,
                                             draw=lrta.PhiloxDraws(seed), canonical=True)
        assert got32.dtype == np.float32
        assert _rel(got32, ref32) <= 1e-4, _rel(got32, ref32)


def _lowrank(dims, r, noise, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((r,) * len(dims))
    for k, n in enumerate(dims):
        x = np.moveaxis(np.tensordot(rng.standard_normal((n, r)), x, axes=([1], [k])), 0, k)
    return x + noise * rng.standard_normal(dims)


@pytest.mark.parametrize("dims,r,eps,block", [
    ((128, 512, 64), 6, 0.1, 8),     # n = 32768: two-level TSQR of the n x b blocks
    ((96, 80, 12), 12, 0.05, 10),    # several bidiagonalisation steps per mode
])
def test_blbp_larger_matches_oracle(cuda_lib, dims, r, eps, block):
    import paper_2506_09594_b200 as pk

    a = _lowrank(dims, r, 0.05, 3)
    tf, diag = pk.ad_rsthosvd_blbp(a, eps, block=block, order=(0, 1), seed=4)
    core, factors, od = lrta.ad_rsthosvd_blbp(a, eps, block, None, (0, 1),
                                              draw=lrta.PhiloxDraws(4), canonical=True)
    for k in (0, 1):
        assert diag.ranks[k] == od["ranks"][k] and diag.iterations[k] == od["iterations"][k]
        assert _rel(tf.factors[k], factors[k]) <= 1e-9
    assert _rel(tf.core, core) <= 1e-9
    sk = pk.SketchConfig(mode="fixed-accuracy", eps=eps, block=block, seed=4)
    got = pk.gnhtsvt_randomized(a, pk.Transform.fft(), pk.MCP(2.5), 0.5, sk)
    ref = lrta.gnhtsvt_randomized_blbp(a, TransformSpec("fft"), MCP, 0.5, eps, block, None,
                                       (0, 1), draw=lrta.PhiloxDraws(4), canonical=True)
    assert _rel(got, ref) <= 1e-9


@pytest.mark.parametrize("i", range(3))
def test_other_orders_match_oracle(cuda_lib, golden, i):
    import paper_2506_09594_b200 as pk

    pre = f"ord{i}_"
    a = golden[pre + "in"]
    order = tuple(int(k) for k in golden[pre + "order"])
    ranks = tuple(int(r) for r in golden[pre + "ranks"])
    blocks = tuple(int(b) for b in golden[pre + "blocks"])
    seed = int(golden[pre + "seed"])
    src = philox.PhiloxSketchSource(seed)
    core, factors = lrta.rsthosvd_bki(a, ranks, order, blocks, None, src, canonical=True)
    # the reference default order (all modes) when the golden case used it
    kw = {} if order == tuple(range(a.ndim)) else {"order": order}
    tf = pk.rsthosvd_bki(a, ranks, blocks=blocks, seed=seed, strict_rank=False, **kw)
    for k in order:
        assert _rel(tf.factors[k], factors[k]) <= 1e-9, k
    assert _rel(tf.core, core) <= 1e-9
    sk = pk.SketchConfig(mode="fixed-rank", order=order, ranks=ranks, blocks=blocks, seed=seed)
    got = pk.gnhtsvt_randomized(a, pk.Transform.fft(), pk.MCP(2.5), 0.3, sk)
    ref = lrta.gnhtsvt_randomized(a, TransformSpec("fft"), MCP, 0.3, ranks, blocks, None, order,
                                  src, canonical=True)
    assert _rel(got, ref) <= 1e-9, _rel(got, ref)


def test_zero_input_gives_rank_zero(cuda_lib):
    import paper_2506_09594_b200 as pk

    x = np.zeros((8, 7, 5))
    tf = pk.rsthosvd_bki(x, (3, 3), order=(0, 1), blocks=(1, 1), krylov=(2, 2))
    assert tf.ranks == (0, 0, 5) and tf.core.shape == (0, 0, 5)
    assert tf.factors[0].shape == (8, 0) and tf.factors[1].shape == (7, 0)
    assert not tf.reconstruct().any()
    tf2, diag = pk.ad_rsthosvd_blbp(x, 0.1, block=3)
    assert tf2.ranks == (0, 0, 0) and diag.iterations == {0: 0, 1: 0, 2: 0}
    sk = pk.SketchConfig(mode="fixed-accuracy", eps=0.1, block=3)
    assert not pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.MCP(2.5), 0.1, sk).any()


def test_blbp_inside_admm_matches_oracle(cuda_lib, golden):
    """GNRHTC with a fixed-accuracy sketch: every t-SVT runs the block Lanczos
    compression on the GPU (solvers.py:193-196 -> sketch.py:406-427)."""
    import paper_2506_09594_b200 as pk
    from oracle import admm

    mobs, mask = golden["admm_mobs"], golden["admm_mask"]
    sk = pk.SketchConfig(mode="fixed-accuracy", eps=0.05, block=3, seed=2)
    cfg = pk.SolverConfig(max_iters=6, randomized=True, sketch=sk)
    l, e, rep = pk.gnrhtc(mobs, mask, cfg)

    def thr(x, tau):
        return lrta.gnhtsvt_randomized_blbp(x, TransformSpec("fft"), MCP, tau, 0.05, 3, None,
                                            (0, 1), draw=lrta.PhiloxDraws(2), canonical=True)

    lo, eo, hist = admm.admm_complete(mobs, mask, thr, MCP, admm.default_lambda(mobs.shape),
                                      (0, 1, 2), max_iters=6)
    assert _rel(l, lo) <= 1e-9, _rel(l, lo)
    assert _rel(e, eo) <= 1e-9
    np.testing.assert_allclose(np.array(rep.residual_history), np.array(hist["residuals"]),
                               rtol=1e-6, atol=1e-9)
