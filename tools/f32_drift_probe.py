"""Locate the fp32 drift of the rank-(8, 8) randomized GNRHTC case
(tests/test_admm_gpu.py::test_larger_randomized_power_of_two): run the fp32
solver under each fast-path switch and print the error vs the fp64 oracle."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2506_09594_b200 as pk
from test_admm_gpu import _lowrank_problem, _oracle_rnd
mobs, mask = _lowrank_problem()
out = []
for ranks in [(4, 4), (8, 8)]:
    lo, eo, hist = _oracle_rnd(mobs, mask, 6, ranks, (2, 2), (3, 3), 1)
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=ranks, blocks=(2, 2), krylov=(3, 3), seed=1)
    for it in (1, 2, 3, 6):
        lo_i, _, _ = _oracle_rnd(mobs, mask, it, ranks, (2, 2), (3, 3), 1)
        cfg = pk.SolverConfig(max_iters=it, randomized=True, sketch=sk)
        l32, _, _ = pk.gnrhtc(mobs.astype(np.float32), mask, cfg)
        out.append(f"{ranks} it={it} {np.linalg.norm(l32 - lo_i) / np.linalg.norm(lo_i):.3e}")
print(" | ".join(out))
''' % (ROOT, os.path.join(ROOT, "tests"))

for env in ["", "TR_NO_TC", "TR_NO_PANEL_MMA", "TR_NO_ORTH_CLUSTER", "TR_NO_RITZ_APPLY",
            "TR_NO_FUSE", "TR_FFT_SIMPLE", "TR_NO_PANEL"]:
    e = dict(os.environ)
    if env:
        e[env] = "1"
    r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
    print(env or "default", "->", r.stdout.strip() or r.stderr[-400:], flush=True)
