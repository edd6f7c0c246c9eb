"""Parity of the device gradient-system solve (tr_gradsys_*) with the reference.

The reference's own outputs (tests/golden: solve_out, solve2_out) pin the small
odd/even shapes; larger shapes are checked against the oracle restatement of
solve_grad_system (oracle/admm.py, gradient.py:90-106) and cover every
specialised FFT tile kernel (2^7 .. 2^11-point lines), the runtime-shaped
power-of-two kernel, the generic mixed-radix kernel and the full-spectrum path
(odd first axis).
"""

import numpy as np
import pytest

from oracle import admm

pytestmark = pytest.mark.gpu


def test_golden_solves(cuda_lib, golden):
    import paper_2506_09594_b200 as pk
    gm = {k: golden[f"solve_g{k}"] for k in (0, 1, 2)}
    out = pk.solve_grad_system(golden["solve_b"], gm, pk.GradientSet(golden["solve_b"].shape, (0, 1, 2)))
    np.testing.assert_allclose(out, golden["solve_out"], atol=1e-10, rtol=0)
    gm2 = {0: golden["solve2_g0"], 3: golden["solve2_g3"]}
    b2 = golden["solve2_b"]
    out2 = pk.solve_grad_system(b2, gm2, pk.GradientSet(b2.shape, (0, 3)))
    np.testing.assert_allclose(out2, golden["solve2_out"], atol=1e-10, rtol=0)


SHAPES = [
    ((256, 256, 128), (0, 1, 2)),   # R2C 2^7 x16 lines, C2C 2^8 x8 contiguous, 2^7 x16 strided
    ((1024, 64, 8), (0, 2)),        # R2C 2^9 x4
    ((2048, 16, 4), (1, 2)),        # R2C 2^10 x2
    ((4096, 8, 4), (0, 1, 2)),      # R2C 2^11 x1
    ((16, 2048, 3), (1,)),          # C2C 2^11 contiguous, generic half-spectrum pass
    ((32, 1024, 6), (0, 1, 2)),     # C2C 2^10 contiguous, mixed-radix axis 2
    ((64, 24, 40), (0, 1, 2)),      # non power-of-two spectrum axes
    ((31, 16, 4), (0, 1, 2)),       # odd first axis: full complex spectrum
    ((32, 16, 8, 4), (1, 3)),       # order 4
]


@pytest.mark.parametrize("dims,modes", SHAPES)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_solve_matches_oracle(cuda_lib, dims, modes, dt):
    import torch

    import paper_2506_09594_b200 as pk
    rng = np.random.default_rng(hash((dims, modes)) % 2**32)
    b = rng.standard_normal(dims)
    gm = {k: rng.standard_normal(dims) for k in modes}
    ref = admm.solve_grad_system(b, gm, modes)
    gs = pk.GradientSet(dims, modes)
    if dt == "f64":
        out = pk.solve_grad_system(b, gm, gs)
        tol = 1e-9
    else:
        tb = torch.from_numpy(b).float().cuda()
        tg = {k: torch.from_numpy(v).float().cuda() for k, v in gm.items()}
        out = pk.solve_grad_system(tb, tg, gs).double().cpu().numpy()
        tol = 1e-4
    err = np.abs(out - ref).max() / np.abs(ref).max()
    assert err < tol, f"max rel error {err:.3e}"


def test_solve_inverts_operator(cuda_lib):
    """Size-independent property at a bench-scale shape: applying the operator
    to the solution recovers the rhs (gradient.py:82-87)."""
    import paper_2506_09594_b200 as pk
    dims, modes = (512, 256, 64), (0, 1, 2)
    rng = np.random.default_rng(7)
    b = rng.standard_normal(dims)
    x = pk.solve_grad_system(b, {k: np.zeros(dims) for k in modes}, pk.GradientSet(dims, modes))
    np.testing.assert_allclose(admm.apply_operator(x, modes), b, atol=1e-9)


def test_input_errors(cuda_lib):
    import paper_2506_09594_b200 as pk
    with pytest.raises(ValueError):
        pk.GradientSet((8, 8, 8), ())
    with pytest.raises(ValueError):
        pk.GradientSet((8, 8, 8), (3,))
    gs = pk.GradientSet((8, 8, 8), (0,))
    with pytest.raises(ValueError):
        pk.solve_grad_system(np.zeros((8, 8, 4)), {0: np.zeros((8, 8, 4))}, gs)
    with pytest.raises(ValueError):
        pk.solve_grad_system(np.zeros((8, 8, 8)), {0: np.zeros((8, 8, 4))}, gs)
