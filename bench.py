#!/usr/bin/env python
"""Benchmark of the B200 randomized t-SVT hot path ("Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--step lrta|admm]

Workload (BASELINE.json configs[1]): order-3 robust tensor PCA, 1024x1024x128
float32, tubal rank 20 from Gaussian factors, 10% sparse outliers uniform in
[-1, 1]; randomized LRTA target rank 25, Krylov depth q=3, block b=ceil(25/4)=7.

A step (``--step lrta``) is one randomized t-SVT (tenrec.sketch.gnhtsvt_randomized)
of the whole tensor, inputs resident in HBM.  Metric: t-SVT voxels/s (whole job).
The 512 MB tensor exceeds the 126 MB L2, so no explicit flush is needed.

Multi-GPU: one process per GPU (torchrun); every rank runs the step on its own
tensor (independent problems, weak scaling, no data-path collective); the time
is the max over ranks.  ``--impl reference`` times the CPU oracle port of the
reference algorithm on the host cores instead (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = {
    "workload": "rtpca-1024x1024x128-f32",
    "dims": (1024, 1024, 128),
    "tubal_rank": 20,
    "outlier_frac": 0.10,
    "ranks": (25, 25),
    "blocks": (7, 7),
    "krylov": (3, 3),
    "penalty": "mcp(gamma=2.5)",
    "transform": "fft",
}
METRIC = "randomized t-SVT voxels/s"
UNIT = "voxels/s"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(torch, dims, seed):
    """Low-tubal-rank tensor (t-product of Gaussian factors, unit RMS) + outliers.

    Column-major on the device as a flat buffer (the package's layout).  Data
    generation is setup, not part of the timed region.
    """
    n1, n2, n3 = dims
    r = WORKLOAD["tubal_rank"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((n3, r, n1), generator=g, device="cuda", dtype=torch.float32)
    b = torch.randn((n3, n2, r), generator=g, device="cuda", dtype=torch.float32)
    fa = torch.fft.rfft(a, dim=0)
    fb = torch.fft.rfft(b, dim=0)
    # face-wise products in the transform domain: X_f = A_f B_f  ->  (n3, n2, n1)
    fx = torch.einsum("fjk,fki->fji", fb, fa)
    x = torch.fft.irfft(fx, n=n3, dim=0)
    x = x / x.pow(2).mean().sqrt()
    n = x.numel()
    flat = x.reshape(-1)
    k = int(round(WORKLOAD["outlier_frac"] * n))
    idx = torch.randperm(n, generator=g, device="cuda")[:k]
    flat[idx] = torch.rand(k, generator=g, device="cuda") * 2 - 1
    return flat.contiguous()


def algorithmic_bytes(shape, esize):
    """Bytes each kernel category must move per LRTA (per-unit traffic)."""
    n1, n2, n3 = shape
    r0, r1 = WORKLOAD["ranks"]
    b0, b1 = WORKLOAD["blocks"]
    q0, q1 = WORKLOAD["krylov"]
    a0 = n1 * n2 * n3 * esize            # mode-0 unfolding = the tensor
    a1 = n2 * r0 * n3 * esize            # mode-1 unfolding of the mode-0 core
    s0, s1 = (q0 + 1) * b0, (q1 + 1) * b1
    return {
        # one read of the unfolding per sketch / power (+ per-split partial sums)
        "rank_update": (q0 + 1) * a0 + (q1 + 1) * a1,
        # one read per power and per projection, plus the W / coefficient writes
        "dot_cols": (q0 + 1) * a0 + (q1 + 1) * a1 + (n2 * n3 * (q0 * b0 + s0)
                                                     + r0 * n3 * (q1 * b1 + s1)) * esize,
        # write of the reconstructed tensor + read of the expanded core
        "gemm_expand": a0 + r0 * n2 * n3 * esize,
    }


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200 import _lib
    from paper_2506_09594_b200.sketch import _run_lrta
    from paper_2506_09594_b200.tensors import ColMajor

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.lib()
    dims = WORKLOAD["dims"]
    flat = make_workload(torch, dims, 1234 + rank)
    x = ColMajor(flat, dims, "torch", None)
    out = ColMajor(torch.empty_like(flat), dims, "torch", None)
    pen = pk.MCP(2.5)
    tau = 0.05 * float(flat.norm()) / math.sqrt(flat.numel())
    tf = pk.Transform.fft()

    def step():
        _run_lrta(x, out, WORKLOAD["ranks"], WORKLOAD["blocks"], WORKLOAD["krylov"], 7, tf, pen,
                  tau)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = lib.tr_launch_count()
    lib.tr_profile_enable(1)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.tr_launch_count() - launches0
    prof = _lib.profile_read()
    lib.tr_profile_enable(0)
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    voxels = math.prod(dims)
    value = voxels * args.steps * world / (ms / 1e3)

    # end-to-end through the public API with host buffers (H2D + D2H inside)
    host = flat.reshape(tuple(reversed(dims))).permute(2, 1, 0).cpu().numpy()
    host = np.ascontiguousarray(host)
    sk = pk.SketchConfig(mode="fixed-rank", ranks=WORKLOAD["ranks"], blocks=WORKLOAD["blocks"],
                         krylov=WORKLOAD["krylov"], seed=7)
    pk.gnhtsvt_randomized(host, tf, pen, tau, sk)
    e2e_steps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = pk.gnhtsvt_randomized(host, tf, pen, tau, sk)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": voxels / e2e_s, "unit": UNIT, "h2d_bytes_per_step": host.nbytes,
           "d2h_bytes_per_step": res.nbytes, "api": "paper_2506_09594_b200.gnhtsvt_randomized(numpy)"}

    # roofline of the dominant kernel category
    peak, peak_kind = peaks()
    algo = algorithmic_bytes(dims, 4)
    cats = {k: v for k, v in prof.items() if k in algo}
    dom = max(cats, key=lambda k: cats[k][0]) if cats else None
    roof = None
    if dom:
        tot_ms, n_launch = cats[dom]
        per_step_ms = tot_ms / args.steps
        achieved = algo[dom] / (per_step_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "share_of_step": round(per_step_ms / ms_per_step, 4),
                "launches_per_step": n_launch / args.steps}
    breakdown = {k: round(v[0] / args.steps, 4) for k, v in sorted(prof.items(),
                                                                   key=lambda kv: -kv[1][0])}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian-factor t-product + uniform outliers)",
            "config": {"workload": WORKLOAD["workload"], "step": "lrta", "dims": list(dims),
                       "ranks": list(WORKLOAD["ranks"]), "blocks": list(WORKLOAD["blocks"]),
                       "krylov": list(WORKLOAD["krylov"]), "parallelism": f"replicas{world}",
                       "l2": "input 512 MB > 126 MB L2 (no flush needed)"},
            "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "kernel_ms_per_step": breakdown, "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(flat, dims)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(flat=None, dims=None, nf=32, seed=0):
    """The oracle port (numpy restatement of tenrec) timed on the host cores on a
    bounded sample: one randomized t-SVT of a 1024x1024x``nf`` slab in fp64."""
    import numpy as np

    from oracle import lrta, philox
    from oracle.tensor_ops import TransformSpec

    n1, n2, _ = WORKLOAD["dims"]
    if flat is not None:
        x = flat.reshape(tuple(reversed(dims))).permute(2, 1, 0)[:, :, :nf].double().cpu().numpy()
    else:
        x = np.random.default_rng(seed).standard_normal((n1, n2, nf))
    t0 = time.perf_counter()
    lrta.gnhtsvt_randomized(x, TransformSpec("fft"), (2, 2.5, 0.0), 0.05, WORKLOAD["ranks"],
                            WORKLOAD["blocks"], WORKLOAD["krylov"], (0, 1),
                            philox.PhiloxSketchSource(7))
    dt = time.perf_counter() - t0
    return {"value": x.size / dt, "unit": UNIT, "cores": _threads(), "kind": "port",
            "sample": f"one randomized t-SVT of a {n1}x{n2}x{nf} slab (fp64 numpy oracle)",
            "seconds": dt}


def run_reference(args):
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_baseline(nf=16)
    vals, secs = [], 0.0
    for s in range(args.steps):
        r = cpu_baseline(nf=16, seed=s)
        vals.append(r["value"])
        secs += r["seconds"]
    value = statistics.mean(vals)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian)", "impl": "reference",
        "config": {"workload": WORKLOAD["workload"], "step": "lrta",
                   "sample": "1024x1024x16 slab per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _threads(), "kind": "port",
                         "sample": "one randomized t-SVT of a 1024x1024x16 slab per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--step", choices=("lrta",), default="lrta")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
