import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_09594_b200 as pk
from oracle import admm, lrta, philox
from oracle.tensor_ops import TransformSpec, mode_product
rng = np.random.default_rng(5)
core = rng.standard_normal((4, 4, 16))
x = mode_product(mode_product(core, rng.standard_normal((64, 4)), 0), rng.standard_normal((64, 4)), 1)
mask = rng.random(x.shape) < 0.7
mobs = np.where(mask, x, 0.0)
sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(8, 8), blocks=(2, 2), krylov=(3, 3), seed=1)
spec = TransformSpec("fft"); mcp = (2, 2.5, 0.0)
def thr(a, tau):
    return lrta.gnhtsvt_randomized(a, spec, mcp, tau, (8, 8), (2, 2), (3, 3), (0, 1), philox.PhiloxSketchSource(1), canonical=True)
for it in (1, 2, 3, 6):
    cfg = pk.SolverConfig(max_iters=it, randomized=True, sketch=sk)
    lo, eo, h = admm.admm_complete(mobs, mask, thr, mcp, admm.default_lambda(mobs.shape), (0, 1, 2), max_iters=it)
    l64, _, _ = pk.gnrhtc(mobs, mask, cfg)
    l32, _, _ = pk.gnrhtc(mobs.astype(np.float32), mask, cfg)
    n = np.linalg.norm(lo)
    print(it, "f64", np.linalg.norm(l64 - lo) / n, "f32", np.linalg.norm(l32 - lo) / n, "||L||", n)
# single LRTA at this shape in fp32
a = rng.standard_normal((64, 64, 16)) * 3
for tau in (0.0, 5.0, 50.0):
    ref = lrta.gnhtsvt_randomized(a, spec, mcp, tau, (8, 8), (2, 2), (3, 3), (0, 1), philox.PhiloxSketchSource(1))
    g = pk.gnhtsvt_randomized(a.astype(np.float32), pk.Transform.fft(), pk.MCP(), tau, sk)
    print("lrta tau", tau, np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30))
