"""Per-stream launch timeline of one ADMM sweep on the bench workload.

python tools/timeline.py [sweeps]
Launch start / end come from the CUDA events tr::launch records on each
launch's own stream (concurrent streams, not serialised as under ncu).
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
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
for _ in range(n):
    run.step()
torch.cuda.synchronize()
N = 4096
names = ctypes.create_string_buffer(1 << 17)
t0, t1 = (ctypes.c_double * N)(), (ctypes.c_double * N)()
st = (ctypes.c_int64 * N)()
k = lib.tr_profile_timeline(names, 1 << 17, t0, t1, st, N)
cats = names.value.decode().split("\n")[:k]
lib.tr_profile_enable(0)
recs = [(cats[i], t0[i], t1[i], st[i]) for i in range(k)]
streams = sorted(set(r[3] for r in recs), key=lambda s: min(r[1] for r in recs if r[3] == s))
end = max(r[2] for r in recs)
print(f"{k} launches, {end:.3f} ms for {n} sweep(s); streams {len(streams)}")
for si, s in enumerate(streams):
    rs = [r for r in recs if r[3] == s]
    busy = sum(r[2] - r[1] for r in rs)
    print(f"\n== stream {si}: {len(rs)} launches, busy {busy:.3f} ms, span {rs[0][1]:.3f}-{rs[-1][2]:.3f}")
    prev = None
    line = []
    for c, a, b, _ in rs:
        gap = a - prev if prev is not None else 0.0
        if line and line[-1][0] == c and gap < 0.005:
            line[-1][2] += b - a
            line[-1][3] += 1
        else:
            line.append([c, a, b - a, 1, gap])
        prev = b
    for c, a, d, cnt, gap in line:
        g = f" (+{gap * 1e3:.0f}us gap)" if gap > 0.003 else ""
        print(f"   {a:7.3f}  {c:16s} x{cnt:<3d} {d * 1e3:7.1f} us{g}")
run.close()
