"""Phase breakdown of one public-API solve (bench.py's e2e leg) under cProfile.

python tools/e2e_profile.py [n3]   -- 1024 x 1024 x n3 float32, 10 sweeps
"""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09594_b200 as pk  # noqa: E402

n3 = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dims = (1024, 1024, n3)
rng = np.random.default_rng(0)
host = np.asfortranarray(rng.standard_normal(dims, dtype=np.float32))
mask = np.ones(dims, dtype=bool)
sk = pk.SketchConfig(ranks=(25, 25), blocks=(7, 7), krylov=(3, 3), seed=1)
cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk, max_iters=10,
                      tol=1e-30)
for call in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if call == 2:
        pr = cProfile.Profile()
        pr.enable()
    l, e, rep = pk.gnrhtc(host, mask, cfg)
    if call == 2:
        pr.disable()
    print(f"call {call}: {time.perf_counter() - t0:.3f} s, {rep.iterations} iters", flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
