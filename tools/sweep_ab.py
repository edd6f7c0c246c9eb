"""A/B timing of the bench ADMM sweep under environment switches.

python tools/sweep_ab.py [sweeps] [ENV=VAL ...]   (each variant in its own process)
Prints ms per sweep (CUDA events on the solver's main stream, 3 warm-up sweeps,
no profiling events) for the default build and for every listed variant.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
import bench, paper_2506_09594_b200 as pk
from paper_2506_09594_b200 import _lib
from paper_2506_09594_b200.solvers import NativeSolver
from paper_2506_09594_b200.tensors import ColMajor
n = int(sys.argv[1])
dims = bench.WORKLOAD["dims"]
lib = _lib.lib()
flat = bench.make_workload(torch, dims, 1234)
cm = ColMajor(flat, dims, "torch", None)
mask = torch.ones(flat.numel(), dtype=torch.uint8, device="cuda")
sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=bench.WORKLOAD["ranks"],
                     blocks=bench.WORKLOAD["blocks"], krylov=bench.WORKLOAD["krylov"], seed=7)
cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk, tol=1e-30)
run = NativeSolver("gnrhtc", cm, None, mask, cfg, bench.WORKLOAD["modes"], cfg.lam_for(dims))
st = torch.cuda.ExternalStream(lib.tr_admm_stream(run.handle))
for _ in range(3):
    run.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(n):
    run.step()
e1.record(st)
torch.cuda.synchronize()
print("%%.3f" %% (e0.elapsed_time(e1) / n))
''' % ROOT

n = sys.argv[1] if len(sys.argv) > 1 else "20"
variants = [""] + sys.argv[2:]
for v in variants:
    env = dict(os.environ)
    for kv in filter(None, v.split(",")):
        k, _, val = kv.partition("=")
        env[k] = val or "1"
    r = subprocess.run([sys.executable, "-c", CHILD, n], env=env, capture_output=True, text=True)
    print(f"{v or 'default':40s} {r.stdout.strip() or r.stderr[-300:]} ms/sweep", flush=True)
