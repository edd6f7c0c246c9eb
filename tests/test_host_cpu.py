"""CPU-only checks: the C ABI library loads and exports what include/*.h
declares; host-side validation mirrors the reference's errors."""

import os
import re

import numpy as np
import pytest

from paper_2506_09594_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            text = open(os.path.join(inc, fn)).read()
            names |= set(re.findall(r"\b(tr_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert lib.tr_version() >= 100


def test_workspace_query_without_gpu():
    lib = _lib.load()
    ws = lib.tr_lrta_workspace(_lib.F32, 3, _lib.i64([1024, 1024, 128]), _lib.i64([25, 25]),
                               _lib.i64([7, 7]), _lib.i64([3, 3]))
    assert 0 < ws < 2 ** 31
    bad = lib.tr_lrta_workspace(_lib.F32, 3, _lib.i64([10, 10, 4]), _lib.i64([20, 5]),
                                _lib.i64([5, 2]), _lib.i64([3, 3]))
    assert bad == -1
    assert b"out of range" in lib.tr_last_error()


def test_sketch_config_validation_mirrors_reference():
    from paper_2506_09594_b200 import SketchConfig
    with pytest.raises(ValueError, match="requires target ranks"):
        SketchConfig().validate((5, 5, 5))
    with pytest.raises(ValueError, match=r"\(q\+1\)\*b"):
        SketchConfig(ranks=(10, 9), krylov=(2, 2), order=(0, 1)).validate((40, 36, 8))
    with pytest.raises(ValueError, match="exceeds"):
        SketchConfig(ranks=(50, 4), order=(0, 1)).validate((40, 36, 8))
    with pytest.raises(ValueError, match="unknown sketch mode"):
        SketchConfig(mode="x").validate((4, 4, 4))
    with pytest.raises(ValueError, match="eps"):
        SketchConfig(mode="fixed-accuracy", eps=1.5).validate((4, 4, 4))
    SketchConfig(ranks=(10, 9), krylov=(3, 3), order=(0, 1)).validate((40, 36, 8))


def test_penalty_validation_and_factory():
    import paper_2506_09594_b200 as pk
    for bad in (lambda: pk.MCP(gamma=1.0), lambda: pk.Firm(gamma=0.5), lambda: pk.SCAD(a=2.0),
                lambda: pk.Lq(q=0.0), lambda: pk.CappedLq(theta=0.0),
                lambda: pk.LogPenalty(gamma=0.0)):
        with pytest.raises(ValueError):
            bad()
    assert isinstance(pk.make_penalty("capped-lq", q=0.7), pk.CappedLq)
    with pytest.raises(ValueError):
        pk.make_penalty("huber")
    assert pk.MCP(3.0).encode() == (2, 3.0, 0.0)
    assert pk.CappedLq(0.5, 2.0).encode() == (5, 0.5, 2.0)


def test_penalty_values_match_oracle(golden):
    import paper_2506_09594_b200 as pk
    from oracle import prox as P
    pens = {"l1": pk.L1(), "firm": pk.Firm(2.5), "mcp": pk.MCP(2.0), "scad": pk.SCAD(3.7),
            "lq": pk.Lq(0.5), "capped-lq": pk.CappedLq(0.5, 1.0), "log": pk.LogPenalty(1.0)}
    for name, pen in pens.items():
        kind, p0, p1 = pen.encode()
        for mu, v in zip(golden["prox_mu"][:8], golden["prox_v"][:8]):
            np.testing.assert_allclose(pen.value(np.abs(v), mu), P.value(kind, p0, p1, np.abs(v), mu),
                                       rtol=1e-13)


def test_transform_validation():
    import paper_2506_09594_b200 as pk
    rng = np.random.default_rng(5)
    with pytest.raises(pk.TransformError):
        pk.Transform.explicit([rng.standard_normal((4, 4))])
    with pytest.raises(pk.TransformError):
        pk.Transform.explicit([rng.standard_normal((4, 3))])
    t = pk.Transform.explicit([np.eye(4)])
    with pytest.raises(pk.TransformError):
        t.check_shape((3, 3, 5))
    assert pk.Transform.fft().rho((3, 4, 5, 6)) == 30.0
    assert pk.Transform.dct().rho((3, 4, 5)) == 1.0


def test_gpu_entry_points_fail_loudly_without_gpu():
    import torch

    import paper_2506_09594_b200 as pk
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sk = pk.SketchConfig(ranks=(2, 2), blocks=(1, 1), krylov=(2, 2))
    with pytest.raises(_lib.CudaPathError):
        pk.gnhtsvt_randomized(np.ones((4, 4, 3)), pk.Transform.fft(), pk.MCP(), 0.1, sk)
    with pytest.raises(_lib.CudaPathError):
        pk.MCP().prox(1.0, 2.0)
