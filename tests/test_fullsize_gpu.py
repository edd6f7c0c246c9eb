"""Randomized t-SVT parity at BASELINE.json's full shapes (size-independent property).

For X = G x_0 U x_1 V with orthonormal U (n1 x r0), V (n2 x r1) and a random
core G, the transform acts along modes >= 2 only, so every transform-domain
face of X is U G_f V^T and its SVT is U SVT(G_f) V^T:

    gnhtsvt(X) = gnhtsvt(G) x_0 U x_1 V      (tenrec/shrink.py:76-106)

and a randomized Tucker sketch whose ranks cover (r0, r1) captures range(U)
and range(V) exactly (tenrec/sketch.py:211-270), so gnhtsvt_randomized(X)
equals it too.  The right-hand side needs only the oracle's deterministic
GNHTSVT of the small core, so the GPU path (tensor-core Krylov passes, cluster
basis, Rayleigh-Ritz, face SVT, expansion -- or their large-m fallbacks) is
checked at the bench's own 1024 x 1024 x 128 fp32 shape and at the other
BASELINE configs' shapes.
"""

import numpy as np
import pytest

import paper_2506_09594_b200 as pk
from oracle import lrta
from oracle.tensor_ops import TransformSpec

pytestmark = pytest.mark.gpu

# dims (BASELINE config), true multilinear ranks, sketch ranks, blocks, krylov, penalty
CASES = [
    ((1024, 1024, 128), (20, 20), (25, 25), (7, 7), (3, 3), "mcp"),  # configs[1]: bench shape
    ((512, 512, 16, 32), (15, 15), (25, 25), (10, 10), (2, 2), "l1"),  # configs[2]: order 4, b > 8
    ((2048, 2048, 64), (10, 10), (15, 15), (5, 5), (2, 2), "mcp"),  # configs[3]: m = 2048
]
# fp64 at the boundary sizes of the fast paths (cluster basis m <= 1024, the
# CUDA-core panel with a chunk width that is not a multiple of its reduction group)
CASES64 = [
    ((1024, 512, 8), (10, 10), (15, 15), (5, 5), (2, 2), "mcp"),
    ((1056, 512, 8), (10, 10), (15, 15), (5, 5), (2, 2), "l1"),
]


def _penalty(name):
    return {"mcp": (pk.MCP(2.0), (2, 2.0, 0.0)), "l1": (pk.L1(), (0, 0.0, 0.0))}[name]


@pytest.mark.parametrize("case", [(c, "f32") for c in CASES] + [(c, "f64") for c in CASES64],
                         ids=lambda c: "x".join(map(str, c[0][0])) + "-" + c[1])
def test_randomized_tsvt_fullsize_lowrank(case):
    import torch

    (dims, (r0, r1), ranks, blocks, krylov, pname), dt = case
    dtype = torch.float32 if dt == "f32" else torch.float64
    rest = dims[2:]
    g = torch.Generator(device="cuda").manual_seed(11)
    u = torch.linalg.qr(torch.randn(dims[0], r0, generator=g, device="cuda",
                                    dtype=torch.float64))[0]
    v = torch.linalg.qr(torch.randn(dims[1], r1, generator=g, device="cuda",
                                    dtype=torch.float64))[0]
    core = torch.randn((r0, r1) + rest, generator=g, device="cuda", dtype=torch.float64)
    x = torch.einsum("ia,jb,ab...->ij...", u, v, core)
    scale = float(x.abs().max())
    x = (x / scale).to(dtype)
    core = core / scale
    pen, pen_o = _penalty(pname)
    # about the median transform-domain singular value of the core faces
    tau = 0.5 * float(core.std()) * float(np.sqrt(np.prod(rest) * r0))

    sk = pk.SketchConfig(mode="fixed-rank", ranks=ranks, blocks=blocks, krylov=krylov, seed=5)
    got = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pen, tau, sk)
    torch.cuda.synchronize()

    shr = lrta.gnhtsvt(core.cpu().numpy(), TransformSpec("fft"), pen_o, tau)
    want = torch.einsum("ia,jb,ab...->ij...", u, v, torch.as_tensor(shr, device="cuda"))
    got64 = torch.as_tensor(got, device="cuda").to(torch.float64)
    err = float(torch.linalg.norm(got64 - want) / torch.linalg.norm(want))
    # parity bars: 1e-4 for the fp32 stream (fp64 small solves), 1e-9 in fp64
    assert err <= (1e-4 if dt == "f32" else 1e-9), f"rel err {err:.3e}"
    # the threshold really shrank something (not an identity check)
    assert float(torch.linalg.norm(want - x.to(torch.float64))) > 1e-3 * float(
        torch.linalg.norm(want))
