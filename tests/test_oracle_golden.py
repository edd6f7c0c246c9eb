"""Pin the CPU oracle against vectors produced by the reference itself.

The oracle is only trusted as the GPU checker after these pass: every case
below replays a reference call recorded by tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from oracle import admm, lrta, philox
from oracle import prox as P
from oracle.tensor_ops import TransformSpec, unfold

PENS = {"l1": (0, 0.0, 0.0), "firm": (1, 2.5, 0.0), "mcp": (2, 2.0, 0.0), "scad": (3, 3.7, 0.0),
        "lq": (4, 0.5, 0.0), "capped-lq": (5, 0.5, 1.0), "log": (6, 1.0, 0.0)}


@pytest.mark.parametrize("name", sorted(PENS))
def test_prox_and_value_match_reference(golden, name):
    kind, p0, p1 = PENS[name]
    mus, vs = golden["prox_mu"], golden["prox_v"]
    got = np.stack([P.prox(kind, p0, p1, mu, v) for mu, v in zip(mus, vs)])
    np.testing.assert_array_max_ulp(got, golden[f"prox_{name}"], maxulp=4) \
        if name not in ("lq", "capped-lq") else \
        np.testing.assert_allclose(got, golden[f"prox_{name}"], rtol=0, atol=1e-12)
    val = np.stack([P.value(kind, p0, p1, np.abs(v), mu) for mu, v in zip(mus, vs)])
    np.testing.assert_allclose(val, golden[f"value_{name}"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("q", [0.3, 0.7, 1.0])
def test_lq_exponents(golden, q):
    got = np.stack([P.prox(4, q, 0.0, mu, v) for mu, v in zip(golden["prox_mu"], golden["prox_v"])])
    np.testing.assert_allclose(got, golden[f"prox_lq{q}"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("structure", ["entry", "tube", "slice"])
def test_gnhtt(golden, structure):
    got = lrta.gnhtt(golden["gnhtt_in"], PENS["mcp"], 0.9, structure)
    np.testing.assert_allclose(got, golden[f"gnhtt_{structure}"], rtol=0, atol=1e-14)


def test_transforms(golden):
    x = golden["tr_in"]
    specs = {"fft": TransformSpec("fft"), "dct": TransformSpec("dct"),
             "explicit": TransformSpec("explicit", [golden["tr_mat0"], golden["tr_mat1"]])}
    for kind, spec in specs.items():
        np.testing.assert_allclose(spec.apply(x), golden[f"tr_{kind}"], rtol=0, atol=1e-13)
        assert spec.rho(x.shape) == pytest.approx(float(golden[f"tr_{kind}_rho"]), rel=1e-13)
        np.testing.assert_allclose(spec.inverse(spec.apply(x)), x, atol=1e-13)


@pytest.mark.parametrize("i", range(5))
def test_gnhtsvt_deterministic(golden, i):
    a = golden[f"svt{i}_in"]
    pen = PENS[str(golden[f"svt{i}_pen"])]
    tau = float(golden[f"svt{i}_tau"])
    for kind in ("fft", "dct"):
        got = lrta.gnhtsvt(a, TransformSpec(kind), pen, tau)
        np.testing.assert_allclose(got, golden[f"svt{i}_{kind}"], rtol=0, atol=1e-12)


def _rcase(golden, i):
    pre = f"rsvt{i}_"
    return dict(a=golden[pre + "in"], ranks=tuple(golden[pre + "ranks"]),
                blocks=tuple(golden[pre + "blocks"]), krylov=tuple(golden[pre + "krylov"]),
                seed=int(golden[pre + "seed"]), pen=PENS[str(golden[pre + "pen"])],
                tau=float(golden[pre + "tau"]), lowrank=int(golden[pre + "lowrank"]))


@pytest.mark.parametrize("i", range(5))
def test_randomized_exact_reference_stream(golden, i):
    """With the reference's PCG64 draws and its LAPACK sign convention the
    oracle reproduces the reference output and factors."""
    c = _rcase(golden, i)
    src = philox.NumpySketchSource(c["seed"])
    core, fac = lrta.rsthosvd_bki(c["a"], c["ranks"], (0, 1), c["blocks"], c["krylov"], src,
                                  canonical=False)
    pre = f"rsvt{i}_"
    np.testing.assert_allclose(fac[0], golden[pre + "f0"], atol=1e-10)
    np.testing.assert_allclose(fac[1], golden[pre + "f1"], atol=1e-10)
    np.testing.assert_allclose(core, golden[pre + "core"], atol=1e-10 * np.abs(core).max())
    out = lrta.gnhtsvt_randomized(c["a"], TransformSpec("fft"), c["pen"], c["tau"], c["ranks"],
                                  c["blocks"], c["krylov"], (0, 1),
                                  philox.NumpySketchSource(c["seed"]), canonical=False)
    ref = golden[pre + "out"]
    assert np.linalg.norm(out - ref) <= 1e-11 * max(np.linalg.norm(ref), 1.0)


@pytest.mark.parametrize("i", range(5))
def test_randomized_canonical_sign_is_a_column_sign_change(golden, i):
    """Canonical signs change F0 only by column signs; mode-0 is sketch-identical."""
    c = _rcase(golden, i)
    _, fac = lrta.rsthosvd_bki(c["a"], c["ranks"], (0, 1), c["blocks"], c["krylov"],
                               philox.NumpySketchSource(c["seed"]), canonical=True)
    f0 = golden[f"rsvt{i}_f0"]
    np.testing.assert_allclose(np.abs(fac[0].T @ f0), np.eye(f0.shape[1]), atol=1e-8)


@pytest.mark.parametrize("i", [0, 3])
def test_randomized_lowrank_is_sign_invariant(golden, i):
    """On exactly low-rank inputs the canonical-sign oracle, fed either RNG,
    returns the reference output."""
    c = _rcase(golden, i)
    ref = golden[f"rsvt{i}_out"]
    for src in (philox.NumpySketchSource(c["seed"]), philox.PhiloxSketchSource(c["seed"])):
        out = lrta.gnhtsvt_randomized(c["a"], TransformSpec("fft"), c["pen"], c["tau"],
                                      c["ranks"], c["blocks"], c["krylov"], (0, 1), src, True)
        assert np.linalg.norm(out - ref) <= 1e-9 * np.linalg.norm(ref)


def test_reference_draw_order_recorded(golden):
    """The recorded draws are the reference stream: mode 0 then mode 1."""
    c = _rcase(golden, 1)
    src = philox.NumpySketchSource(c["seed"])
    np.testing.assert_array_equal(src.draw(0, *golden["rsvt1_g0"].shape), golden["rsvt1_g0"])
    np.testing.assert_array_equal(src.draw(1, *golden["rsvt1_g1"].shape), golden["rsvt1_g1"])


def test_grad_and_solve(golden):
    b = golden["solve_b"]
    for k in range(3):
        np.testing.assert_array_equal(admm.grad(b, k), golden[f"grad{k}"])
        np.testing.assert_array_equal(admm.grad_adjoint(b, k), golden[f"gradT{k}"])
    gm = {k: golden[f"solve_g{k}"] for k in range(3)}
    np.testing.assert_allclose(admm.solve_grad_system(b, gm, (0, 1, 2)), golden["solve_out"],
                               atol=1e-13)
    gm2 = {0: golden["solve2_g0"], 3: golden["solve2_g3"]}
    np.testing.assert_allclose(admm.solve_grad_system(golden["solve2_b"], gm2, (0, 3)),
                               golden["solve2_out"], atol=1e-13)


def _admm(golden, tag):
    mobs, mask = golden["admm_mobs"], golden["admm_mask"]
    spec = TransformSpec("fft")
    mcp = (2, 2.5, 0.0)
    if tag == "rnd":
        def thr(a, tau):
            return lrta.gnhtsvt_randomized(a, spec, mcp, tau, (6, 5), (2, 2), (2, 2), (0, 1),
                                           philox.NumpySketchSource(3), canonical=False)
    else:
        def thr(a, tau):
            return lrta.gnhtsvt(a, spec, mcp, tau)
    psi = (0, 0.0, 0.0) if tag == "tube" else mcp
    lam = admm.default_lambda(mobs.shape)
    return admm.admm_complete(mobs, mask, thr, psi, lam, (0, 1, 2),
                              structure="tube" if tag == "tube" else "entry", max_iters=15,
                              noise_free=(tag == "nf"), pure_lowrank=(tag == "pure"))


@pytest.mark.parametrize("tag", ["det", "rnd", "tube", "pure", "nf"])
def test_admm_runs(golden, tag):
    l, e, hist = _admm(golden, tag)
    np.testing.assert_allclose(l, golden[f"admm_{tag}_l"], atol=1e-9)
    np.testing.assert_allclose(np.array(hist["residuals"]), golden[f"admm_{tag}_res"],
                               rtol=1e-6, atol=1e-9)
    if tag != "nf":
        np.testing.assert_allclose(e, golden[f"admm_{tag}_e"], atol=1e-9)
        np.testing.assert_allclose(np.array(hist["multipliers"]), golden[f"admm_{tag}_mult"],
                                   rtol=1e-8)


def test_onebit(golden):
    idx, sgn, theta = golden["ob_idx"], golden["ob_sgn"], float(golden["ob_theta"])
    dims = golden["ob_j1"].shape
    j1, j2 = admm.onebit_aggregates(dims, theta, idx, sgn)
    np.testing.assert_array_equal(j1, golden["ob_j1"])
    np.testing.assert_array_equal(j2, golden["ob_j2"])
    spec = TransformSpec("fft")
    mcp = (2, 2.5, 0.0)

    def thr(a, tau):
        return lrta.gnhtsvt(a, spec, mcp, tau)

    lam = admm.default_lambda(dims)
    l, _, hist = admm.onebit_admm(j1, j2, float(idx.size), thr, lam, (0, 1, 2), theta,
                                  max_iters=12)
    np.testing.assert_allclose(l, golden["ob_l"], atol=1e-9)
    np.testing.assert_allclose(np.array(hist["residuals"]), golden["ob_res"], rtol=1e-6, atol=1e-9)
    l, s, hist = admm.onebit_admm(j1, j2, float(idx.size), thr, lam, (0, 1, 2), theta,
                                  psi=(0, 0.0, 0.0), lam2=0.05, robust=True, max_iters=12)
    np.testing.assert_allclose(l, golden["obr_l"], atol=1e-9)
    np.testing.assert_allclose(s, golden["obr_s"], atol=1e-9)


def test_philox_is_deterministic_and_normal():
    g = philox.sketch_matrix(0, 0, 20000, 5)
    np.testing.assert_array_equal(g, philox.sketch_matrix(0, 0, 20000, 5))
    assert abs(g.mean()) < 0.02 and abs(g.std() - 1.0) < 0.02
    assert not np.array_equal(g, philox.sketch_matrix(0, 1, 20000, 5))
    # index semantics: element (c, t) of an (n, b) draw depends only on c*b + t
    np.testing.assert_array_equal(philox.sketch_matrix(9, 2, 7, 3).ravel(),
                                  philox.gaussian_flat(9, 2, np.arange(21)))


def test_unfold_counting_example():
    x = np.arange(1.0, 9.0).reshape((2, 2, 2), order="F")
    assert unfold(x, 0).tolist() == [[1, 3, 5, 7], [2, 4, 6, 8]]


# -- fixed-accuracy block Lanczos and other processing orders -----------------

def _scale(golden, pre):
    return float(np.abs(golden[pre + "in"]).max())


def _blbp_cases(golden):
    return sorted({int(k[4:k.index("_")]) for k in golden if k.startswith("blbp")})


def _order_cases(golden):
    return sorted({int(k[3:k.index("_")]) for k in golden if k.startswith("ord")})


def _blbp_args(golden, i):
    pre = f"blbp{i}_"
    dt = float(golden[pre + "defl_tol"])
    return (golden[pre + "in"], float(golden[pre + "eps"]), int(golden[pre + "block"]),
            None if dt < 0 else dt, tuple(int(k) for k in golden[pre + "order"]),
            int(golden[pre + "seed"]))


@pytest.mark.parametrize("i", range(5))
def test_blbp_matches_reference(golden, i):
    """ad_rsthosvd_blbp (sketch.py:355-403) with the reference's PCG64 draws."""
    a, eps, block, dtol, order, seed = _blbp_args(golden, i)
    pre = f"blbp{i}_"
    core, factors, diag = lrta.ad_rsthosvd_blbp(a, eps, block, dtol, order,
                                                rng=np.random.default_rng(seed))
    np.testing.assert_allclose(core, golden[pre + "core"], rtol=0, atol=1e-8 * _scale(golden, pre))
    for k in order:
        np.testing.assert_allclose(factors[k], golden[pre + f"f{k}"], rtol=0, atol=1e-8 * _scale(golden, pre))
    ks = sorted(order)
    np.testing.assert_array_equal([diag["ranks"][k] for k in ks], golden[pre + "ranks"])
    np.testing.assert_array_equal([diag["iterations"][k] for k in ks], golden[pre + "iterations"])
    np.testing.assert_array_equal([diag["deflations"][k] for k in ks], golden[pre + "deflations"])
    np.testing.assert_allclose([diag["energy"][k] for k in ks], golden[pre + "energy_estimates"],
                               rtol=1e-6, atol=1e-9 * float(np.sum(a * a)))
    if pre + "svt" in golden:
        got = lrta.gnhtsvt_randomized_blbp(a, TransformSpec("fft"), PENS["mcp"], 0.3, eps, block,
                                           dtol, order, rng=np.random.default_rng(seed))
        np.testing.assert_allclose(got, golden[pre + "svt"], rtol=0, atol=1e-8 * _scale(golden, pre))


@pytest.mark.parametrize("i", range(5))
def test_blbp_canonical_is_a_column_sign_change(golden, i):
    """The GPU's sign convention changes the first processed mode's factor by
    column signs only (the bidiagonalisation is equivariant under column sign
    flips of its blocks); later modes see sign-flipped core rows, hence a
    different random start, so they agree with the reference only up to the
    sketch (exactly for an exactly low-rank input, case 1)."""
    a, eps, block, dtol, order, seed = _blbp_args(golden, i)
    pre = f"blbp{i}_"
    core, factors, diag = lrta.ad_rsthosvd_blbp(a, eps, block, dtol, order,
                                                rng=np.random.default_rng(seed), canonical=True)
    k = order[0]
    ref = golden[pre + f"f{k}"]
    sg = np.sign(np.sum(factors[k] * ref, axis=0))
    np.testing.assert_allclose(factors[k], ref * sg, rtol=0, atol=1e-8 * _scale(golden, pre))
    if i == 1:
        got = lrta.gnhtsvt_randomized_blbp(a, TransformSpec("fft"), PENS["mcp"], 0.3, eps, block,
                                           dtol, order, rng=np.random.default_rng(seed),
                                           canonical=True)
        np.testing.assert_allclose(got, golden[pre + "svt"], rtol=0, atol=1e-8 * _scale(golden, pre))


@pytest.mark.parametrize("i", range(3))
def test_other_orders_match_reference(golden, i):
    """rsthosvd_bki / gnhtsvt_randomized with the default (all modes) and other
    processing orders (sketch.py:211-270, 444-451), reference PCG64 draws."""
    pre = f"ord{i}_"
    a = golden[pre + "in"]
    order = tuple(int(k) for k in golden[pre + "order"])
    ranks = tuple(int(r) for r in golden[pre + "ranks"])
    blocks = tuple(int(b) for b in golden[pre + "blocks"])
    seed = int(golden[pre + "seed"])
    core, factors = lrta.rsthosvd_bki(a, ranks, order, blocks, None,
                                      philox.NumpySketchSource(seed), canonical=False)
    np.testing.assert_allclose(core, golden[pre + "core"], rtol=0, atol=1e-8 * _scale(golden, pre))
    for k in order:
        np.testing.assert_allclose(factors[k], golden[pre + f"f{k}"], rtol=0, atol=1e-8 * _scale(golden, pre))
    got = lrta.gnhtsvt_randomized(a, TransformSpec("fft"), PENS["mcp"], 0.3, ranks, blocks, None,
                                  order, philox.NumpySketchSource(seed), canonical=False)
    np.testing.assert_allclose(got, golden[pre + "svt"], rtol=0, atol=1e-8 * _scale(golden, pre))
