import sys, ctypes, math, time
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2506_09594_b200 as pk
from paper_2506_09594_b200 import _lib
from paper_2506_09594_b200.sketch import _run_lrta
from paper_2506_09594_b200.tensors import ColMajor
import bench
lib = _lib.lib()
lib.tr_debug_read.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int]
dbg = (ctypes.c_int * 8)()
dims = (1024, 1024, 128)
flat = bench.make_workload(torch, dims, 1)
x = ColMajor(flat, dims, "torch", None)
out = ColMajor(torch.empty_like(flat), dims, "torch", None)
for tau in (0.0, 0.5, 5.0):
    lib.tr_debug_read(dbg, 1)
    torch.cuda.synchronize(); t = time.time()
    _run_lrta(x, out, (25, 25), (7, 7), (3, 3), 7, pk.Transform.fft(), pk.MCP(2.5), tau)
    torch.cuda.synchronize(); dt = time.time() - t
    lib.tr_debug_read(dbg, 1)
    print("tau", tau, "ritz sweeps (2 calls)", dbg[0], "face sweeps (128 faces)", dbg[1], "ms", dt * 1e3)
