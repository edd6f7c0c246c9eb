"""Dev tool: randomized t-SVT of an exactly low-multilinear-rank tensor against
the oracle's core GNHTSVT (the test_fullsize_gpu property) over a list of shapes.
python tools/bisect_large_m.py [n1 n2 nf dtype]..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09594_b200 as pk  # noqa: E402
from oracle import lrta  # noqa: E402
from oracle.tensor_ops import TransformSpec  # noqa: E402


def run(dims, r, ranks, blocks, krylov, dtype=torch.float32):
    rest = dims[2:]
    g = torch.Generator(device="cuda").manual_seed(11)
    u = torch.linalg.qr(torch.randn(dims[0], r, generator=g, device="cuda", dtype=torch.float64))[0]
    v = torch.linalg.qr(torch.randn(dims[1], r, generator=g, device="cuda", dtype=torch.float64))[0]
    core = torch.randn((r, r) + rest, generator=g, device="cuda", dtype=torch.float64)
    x = torch.einsum("ia,jb,ab...->ij...", u, v, core)
    sc = float(x.abs().max())
    x = (x / sc).to(dtype)
    core = core / sc
    tau = 0.5 * float(core.std()) * float(np.sqrt(np.prod(rest) * r))
    sk = pk.SketchConfig(mode="fixed-rank", ranks=ranks, blocks=blocks, krylov=krylov, seed=5)
    got = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.MCP(2.0), tau, sk)
    torch.cuda.synchronize()
    shr = lrta.gnhtsvt(core.cpu().numpy(), TransformSpec("fft"), (2, 2.0, 0.0), tau)
    want = torch.einsum("ia,jb,ab...->ij...", u, v, torch.as_tensor(shr, device="cuda"))
    got64 = torch.as_tensor(got, device="cuda").to(torch.float64)
    return float(torch.linalg.norm(got64 - want) / torch.linalg.norm(want))


args = sys.argv[1:]
cases = [(tuple(int(v) for v in args[i:i + 3]), args[i + 3]) for i in range(0, len(args), 4)]
for dims, dt in cases:
    t = torch.float32 if dt == "f32" else torch.float64
    print(dims, dt, f"{run(dims, 10, (15, 15), (5, 5), (2, 2), t):.2e}", flush=True)
