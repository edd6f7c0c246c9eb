"""Parity of the CUDA randomized t-SVT against the oracle (and the reference).

Tolerances (north_star): relative error <= 1e-9 in fp64 mode, <= 1e-4 in fp32
mode, oracle and GPU consuming the same Philox sketch stream.
"""

import numpy as np
import pytest

from oracle import lrta, philox
from oracle import prox as P
from oracle.tensor_ops import TransformSpec

pytestmark = pytest.mark.gpu

PENS = {"l1": (0, 0.0, 0.0), "firm": (1, 2.5, 0.0), "mcp": (2, 2.0, 0.0), "scad": (3, 3.7, 0.0),
        "lq": (4, 0.5, 0.0), "capped-lq": (5, 0.5, 1.0), "log": (6, 1.0, 0.0)}


def _pen_obj(name):
    import paper_2506_09594_b200 as pk
    return {"l1": pk.L1(), "firm": pk.Firm(2.5), "mcp": pk.MCP(2.0), "scad": pk.SCAD(3.7),
            "lq": pk.Lq(0.5), "capped-lq": pk.CappedLq(0.5, 1.0), "log": pk.LogPenalty(1.0)}[name]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _tensor(dims, lowrank, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    if not lowrank:
        return rng.standard_normal(dims)
    from oracle.tensor_ops import mode_product
    core = rng.standard_normal((lowrank, lowrank) + tuple(dims[2:]))
    x = mode_product(mode_product(core, rng.standard_normal((dims[0], lowrank)), 0),
                     rng.standard_normal((dims[1], lowrank)), 1)
    return x + noise * rng.standard_normal(dims)


CASES = [
    # dims, ranks, blocks, krylov, lowrank, pen, tau
    ((40, 36, 8), (10, 9), (4, 3), (2, 3), 0, "mcp", 0.5),
    ((33, 29, 7), (8, 8), (3, 2), (3, 3), 0, "l1", 0.3),
    ((24, 20, 4, 3), (6, 6), (2, 3), (3, 2), 0, "scad", 0.2),
    ((64, 48, 6), (12, 10), (4, 5), (2, 1), 8, "lq", 0.4),
    ((50, 60, 5), (16, 12), (4, 4), (3, 2), 0, "capped-lq", 0.3),
    ((30, 28, 9), (7, 6), (2, 2), (3, 3), 0, "log", 0.2),
    ((20, 22, 6), (5, 5), (2, 2), (2, 2), 0, "firm", 0.4),
    # m % 32 == 0 in both modes: fused TMA panel passes + tcgen05 projection
    ((128, 96, 10), (12, 10), (4, 4), (2, 2), 0, "mcp", 0.3),
    # target rank = true rank: ranks above it would pick Ritz vectors in the
    # pure-noise subspace, which are ill-conditioned for any implementation
    ((256, 128, 8), (10, 10), (4, 4), (3, 3), 10, "l1", 0.2),
    ((192, 160, 3, 4), (20, 18), (5, 6), (3, 2), 0, "scad", 0.25),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_gnhtsvt_randomized_matches_oracle(cuda_lib, case, dtype):
    import paper_2506_09594_b200 as pk
    dims, ranks, blocks, krylov, lr, pname, tau = case
    x = _tensor(dims, lr, 3, noise=0.05 if lr else 0.0)
    seed = 17
    ref = lrta.gnhtsvt_randomized(x, TransformSpec("fft"), PENS[pname], tau, ranks, blocks, krylov,
                                  (0, 1), philox.PhiloxSketchSource(seed), canonical=True)
    sk = pk.SketchConfig(mode="fixed-rank", ranks=ranks, blocks=blocks, krylov=krylov, seed=seed)
    xin = x if dtype == "f64" else x.astype(np.float32)
    got = pk.gnhtsvt_randomized(xin, pk.Transform.fft(), _pen_obj(pname), tau, sk)
    assert got.shape == x.shape and got.dtype == xin.dtype
    tol = 1e-9 if dtype == "f64" else 1e-4
    assert _rel(got, ref) <= tol, _rel(got, ref)


@pytest.mark.parametrize("kind", ["dct", "explicit"])
def test_other_transforms(cuda_lib, kind):
    import paper_2506_09594_b200 as pk
    dims = (30, 26, 5, 3)
    x = _tensor(dims, 0, 5)
    rng = np.random.default_rng(9)
    mats = [np.linalg.qr(rng.standard_normal((n, n)))[0] * np.sqrt(1.0 + i)
            for i, n in enumerate(dims[2:])]
    spec = TransformSpec(kind, mats if kind == "explicit" else None)
    tr = pk.Transform.dct() if kind == "dct" else pk.Transform.explicit(mats)
    ref = lrta.gnhtsvt_randomized(x, spec, PENS["mcp"], 0.3, (7, 6), (2, 2), (3, 3), (0, 1),
                                  philox.PhiloxSketchSource(4), canonical=True)
    sk = pk.SketchConfig(ranks=(7, 6), blocks=(2, 2), krylov=(3, 3), seed=4)
    got = pk.gnhtsvt_randomized(x, tr, pk.MCP(2.0), 0.3, sk)
    assert _rel(got, ref) <= 1e-9


def test_factors_and_core_match_oracle(cuda_lib):
    import paper_2506_09594_b200 as pk
    x = _tensor((45, 38, 6), 0, 11)
    core, fac = lrta.rsthosvd_bki(x, (9, 8), (0, 1), (3, 2), (2, 3),
                                  philox.PhiloxSketchSource(5), canonical=True)
    tf = pk.rsthosvd_bki(x, (9, 8), order=(0, 1), blocks=(3, 2), krylov=(2, 3), seed=5)
    np.testing.assert_allclose(tf.factors[0], fac[0], atol=1e-9)
    np.testing.assert_allclose(tf.factors[1], fac[1], atol=1e-9)
    assert _rel(tf.core, core) <= 1e-9


def _golden_case(golden, i):
    pre = f"rsvt{i}_"
    return dict(a=golden[pre + "in"], ranks=tuple(golden[pre + "ranks"]),
                blocks=tuple(golden[pre + "blocks"]), krylov=tuple(golden[pre + "krylov"]),
                seed=int(golden[pre + "seed"]), pen=str(golden[pre + "pen"]),
                tau=float(golden[pre + "tau"]), lowrank=int(golden[pre + "lowrank"]),
                g0=golden[pre + "g0"], g1=golden[pre + "g1"], out=golden[pre + "out"])


@pytest.mark.parametrize("i", range(5))
def test_reference_stream_replay(cuda_lib, golden, i):
    """Fed the reference's own PCG64 draws, the GPU matches the reference on
    exactly low-rank inputs and the canonical-sign oracle everywhere."""
    import paper_2506_09594_b200 as pk
    c = _golden_case(golden, i)
    pen = {"mcp": pk.MCP(2.0), "l1": pk.L1(), "scad": pk.SCAD(3.7)}[c["pen"]]
    sk = pk.SketchConfig(ranks=c["ranks"], blocks=c["blocks"], krylov=c["krylov"], seed=c["seed"])
    got = pk.gnhtsvt_randomized(c["a"], pk.Transform.fft(), pen, c["tau"], sk,
                                sketch_override=(c["g0"], c["g1"]))
    orc = lrta.gnhtsvt_randomized(c["a"], TransformSpec("fft"), PENS[c["pen"]], c["tau"],
                                  c["ranks"], c["blocks"], c["krylov"], (0, 1),
                                  philox.NumpySketchSource(c["seed"]), canonical=True)
    assert _rel(got, orc) <= 1e-9
    if c["lowrank"]:
        assert _rel(got, c["out"]) <= 1e-9


def test_zero_tensor_returns_zero(cuda_lib):
    import paper_2506_09594_b200 as pk
    sk = pk.SketchConfig(ranks=(4, 4), blocks=(2, 2), krylov=(2, 2))
    out = pk.gnhtsvt_randomized(np.zeros((12, 10, 4)), pk.Transform.fft(), pk.MCP(), 0.1, sk)
    assert np.all(out == 0)


@pytest.mark.parametrize("scale", [1e20, 1e-20])
def test_scale_invariance(cuda_lib, scale):
    """The l1 t-SVT is positively homogeneous: the Jacobi rotations of the core
    faces and of the Rayleigh-Ritz Gram (fp32 tangents on operands scaled by a
    power of two) must not depend on the magnitude of the data."""
    import paper_2506_09594_b200 as pk
    x = _tensor((48, 40, 6), 0, 5)
    ref = lrta.gnhtsvt_randomized(x, TransformSpec("fft"), PENS["l1"], 0.4, (9, 8), (3, 3), (2, 2),
                                  (0, 1), philox.PhiloxSketchSource(4), canonical=True)
    sk = pk.SketchConfig(ranks=(9, 8), blocks=(3, 3), krylov=(2, 2), seed=4)
    got = pk.gnhtsvt_randomized(x * scale, pk.Transform.fft(), pk.L1(), 0.4 * scale, sk)
    assert np.all(np.isfinite(got))
    assert _rel(got / scale, ref) <= 1e-9


def test_constant_along_the_transformed_mode(cuda_lib):
    """Identical frontal slices: every transform-domain face but the first is
    (numerically) zero -- tiny faces next to an O(1) one in the face SVT."""
    import paper_2506_09594_b200 as pk
    a = np.random.default_rng(9).standard_normal((40, 36))
    x = np.repeat(a[:, :, None], 8, axis=2)
    ref = lrta.gnhtsvt_randomized(x, TransformSpec("fft"), PENS["mcp"], 0.5, (8, 8), (3, 3), (2, 2),
                                  (0, 1), philox.PhiloxSketchSource(6), canonical=True)
    sk = pk.SketchConfig(ranks=(8, 8), blocks=(3, 3), krylov=(2, 2), seed=6)
    got = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.MCP(2.0), 0.5, sk)
    assert _rel(got, ref) <= 1e-9


def test_deflated_krylov_block(cuda_lib):
    """m < (q+1) b: the Krylov block deflates to rank m, as in the reference."""
    import paper_2506_09594_b200 as pk
    x = _tensor((6, 40, 5), 0, 21)
    ref = lrta.gnhtsvt_randomized(x, TransformSpec("fft"), PENS["mcp"], 0.2, (6, 8), (2, 2),
                                  (3, 3), (0, 1), philox.PhiloxSketchSource(2), canonical=True)
    sk = pk.SketchConfig(ranks=(6, 8), blocks=(2, 2), krylov=(3, 3), seed=2)
    got = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.MCP(2.0), 0.2, sk)
    assert _rel(got, ref) <= 1e-9


def test_tau_zero_is_tucker_projection(cuda_lib):
    import paper_2506_09594_b200 as pk
    x = _tensor((30, 30, 4), 5, 8)
    sk = pk.SketchConfig(ranks=(6, 6), blocks=(2, 2), krylov=(3, 3))
    got = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.L1(), 0.0, sk)
    assert _rel(got, x) <= 1e-9


@pytest.mark.parametrize("name", sorted(PENS))
def test_device_prox_matches_reference(cuda_lib, golden, name):
    import paper_2506_09594_b200 as pk
    pen = _pen_obj(name)
    if name == "mcp":
        pen = pk.MCP(2.0)
    got = np.stack([pen.prox(float(mu), v) for mu, v in zip(golden["prox_mu"], golden["prox_v"])])
    np.testing.assert_allclose(got, golden[f"prox_{name}"], rtol=0, atol=1e-12)
    assert pen.prox(0.0, 2.7) == 2.7 and pen.prox(1.3, 0.0) == 0.0
    kind, p0, p1 = PENS[name]
    v = np.linspace(-6, 6, 101)
    np.testing.assert_allclose(pen.prox(0.8, v), P.prox(kind, p0, p1, 0.8, v), atol=1e-12)
