"""Per-category device time of ADMM sweeps on the bench workload.

TR_SERIAL_MODES=1 python tools/sweep_profile.py [sweeps]
With TR_SERIAL_MODES the per-mode LRTA chains run on one stream, so every
category time is the kernel's own (uncontended) duration.  Also prints the
launch count.
"""

import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_09594_b200 as pk  # noqa: E402
from paper_2506_09594_b200 import _lib  # noqa: E402
from paper_2506_09594_b200.solvers import NativeSolver  # noqa: E402
from paper_2506_09594_b200.tensors import ColMajor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dims = bench.WORKLOAD["dims"]
lib = _lib.lib()
flat = bench.make_workload(torch, dims, 1234)
cm = ColMajor(flat, dims, "torch", None)
mask = torch.ones(flat.numel(), dtype=torch.uint8, device="cuda")
sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=bench.WORKLOAD["ranks"],
                     blocks=bench.WORKLOAD["blocks"], krylov=bench.WORKLOAD["krylov"], seed=7)
cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk, tol=1e-30)
run = NativeSolver("gnrhtc", cm, None, mask, cfg, bench.WORKLOAD["modes"], cfg.lam_for(dims))
for _ in range(3):
    run.step()
torch.cuda.synchronize()
lib.tr_profile_enable(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    run.step()
e1.record()
torch.cuda.synchronize()
prof = _lib.profile_read()
lib.tr_profile_enable(0)
print(f"serial={os.environ.get('TR_SERIAL_MODES') is not None}  ms/sweep {e0.elapsed_time(e1) / n:.3f}")
tot = 0.0
for k, (ms, cnt) in sorted(prof.items(), key=lambda x: -x[1][0]):
    tot += ms / n
    print(f"  {k:18s} {ms / n * 1e3:9.1f} us/sweep  {cnt / n:6.1f} launches/sweep")
run.close()
