"""Per-category kernel time of one configs[4]-shard sweep (bench --step
admm-sharded at N = 1), CUDA events per launch (tr_profile_*)."""
import math
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_09594_b200 as pk  # noqa: E402
from paper_2506_09594_b200 import _lib  # noqa: E402
from paper_2506_09594_b200.shard import DeviceComm, ShardedSolver  # noqa: E402
from paper_2506_09594_b200.tensors import ColMajor  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
lib = _lib.lib()
C = bench.CONFIG4
ld = C["local_dims"]
flat, mask = bench.make_config4_slab(torch, 1, 0)
cm = ColMajor(flat, ld, "torch", None)
sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=C["ranks"], blocks=C["blocks"],
                     krylov=C["krylov"], seed=7)
cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk, tol=1e-30)
run = ShardedSolver("gnrhtc", cm, mask, cfg, (0, 1, 2, 3), cfg.lam_for(ld), ld[-1], 0, DeviceComm())
for _ in range(2):
    run.step()
torch.cuda.synchronize()
lib.tr_profile_enable(1)
run.step()
torch.cuda.synchronize()
import ctypes  # noqa: E402
NMAX = 4096
names = ctypes.create_string_buffer(1 << 17)
t0, t1 = (ctypes.c_double * NMAX)(), (ctypes.c_double * NMAX)()
sts = (ctypes.c_int64 * NMAX)()
n = lib.tr_profile_timeline(names, 1 << 17, t0, t1, sts, NMAX)
cats = names.value.decode().split("\n")
if "--timeline" in sys.argv:
    for i in range(n):
        if cats[i] in ("fft", "orth", "dot_cols"):
            print(f"  {cats[i]:12s} {t0[i]:9.3f} {1e3 * (t1[i] - t0[i]):10.1f} us")
prof = _lib.profile_read()
lib.tr_profile_enable(0)
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:20s} {ms:9.3f} ms  x{n}")
dist.destroy_process_group()
