#!/usr/bin/env python
"""Benchmark of the B200 randomized t-SVT / ADMM hot path ("Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--step admm|lrta|tsvt-sharded|admm-sharded] [--lrta bki|blbp]

Workload (BASELINE.json configs[1]): order-3 robust tensor PCA, 1024x1024x128
float32, tubal rank 20 from Gaussian factors (unit RMS), 10% sparse outliers
uniform in [-1, 1], full observation set; GNRHTC with MCP penalties, gradient
modes {0, 1, 2}, randomized t-SVT of target rank 25, Krylov depth q = 3, block
b = ceil(25/4) = 7.

A step (``--step admm``, default) is one ADMM sweep of tenrec.solvers.gnrhtc:
FFT-diagonal L-solve, three randomized t-SVTs (one per gradient mode), noise /
dual / multiplier updates, Eq. (24) residuals back to the host.  Metric:
randomized t-SVT voxels/s = 3 x 1024*1024*128 x sweeps/s (whole job); ADMM
sweeps/s is reported beside it.  ``--step lrta`` times a single t-SVT;
``--step tsvt-sharded`` times one t-SVT of the whole tensor sharded along its
last mode over the N ranks (strong scaling, NCCL all-reduces of the Krylov
blocks / Ritz Gram / core, shard.py); ``--step admm-sharded`` times one GNRHTC
sweep of BASELINE configs[4]'s tensor sharded along its last mode (global
2048x2048x32x(4N), 4 faces per rank: exactly configs[4] at N = 8; weak
scaling; all-to-all FFT transpose, halo exchanges, sharded t-SVTs).  Every
tensor is 512 MB (> 126 MB L2), so no explicit flush is needed.  The solver
runs with its lookahead on, as the public solvers do (the next sweep's L-solve
is enqueued before the host reads a sweep's residuals): the timed region of K
steps holds exactly K L-solves and K of everything else (the first step's
L-solve was enqueued by the last warm-up step, the K-th step enqueues the next).
The ``roofline`` object is the kernel category with the largest UNCONTENDED
device time per step (the three t-SVT chains of a sweep overlap on concurrent
streams, so their categories are timed in a standalone t-SVT pass).

Multi-GPU: one process per GPU (torchrun); each rank solves its own problem
(independent recoveries, weak scaling, no data-path collective); time = max
over ranks.  ``--impl reference`` times the reference itself (tenrec, installed
into baseline/_ref; the oracle port when absent) on the host cores instead
(rank 0 only): a step is one fp64 GNRHTC sweep of a 1024x1024x4 slab, and one
sweep of the whole bench tensor is timed beside it (``full_config``).
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
    "modes": (0, 1, 2),
    "penalty": "mcp(gamma=2.5) for phi and psi",
    "transform": "fft",
}
METRIC = "randomized t-SVT voxels/s"
UNIT = "voxels/s"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_traffic():
    """DRAM bytes per sweep by kernel category from the newest committed ncu
    capture (profiles/r*/traffic.json), or {}."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")))
    if not files:
        return {}, None
    try:
        with open(files[-1]) as fh:
            t = json.load(fh)
        return t.get("categories", {}), os.path.relpath(files[-1], ROOT)
    except Exception:
        return {}, None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (pynvml) polled from a thread every 2 ms, with one sample forced at
    entry and one at exit so short regions are still covered; nvidia-smi
    (-lms 100) only when NVML is unavailable.
    """

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    BITS = (0x8, 0x40, 0x20, 0x4)  # nvmlClocksEventReason{HwSlowdown,HwThermal,SwThermal,SwPowerCap}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, sm_max_mhz, reasons bitmask)
        self.nv = None
        self.handle = None
        self.thread = None
        self.stop = None
        self.proc = None
        self.source = "none"
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.handle = self._handle(pynvml, index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.source = "nvml"
        except Exception:
            self.nv = None

    @staticmethod
    def _handle(pynvml, index):
        try:
            import torch

            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(index)

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        self.samples.append((float(sm), float(self.smax), int(rs)))

    def _loop(self):
        while not self.stop.wait(0.002):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        import threading

        if self.nv is not None:
            self._sample()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()
            self._sample()
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for ln in out.splitlines():
                parts = [q.strip() for q in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    bits = sum(b for b, v in zip(self.BITS, parts[2:6]) if v.lower() == "active")
                    self.samples.append((float(parts[0]), float(parts[1]), bits))
                except ValueError:
                    continue

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "source": self.source}
        reasons = sorted({nm for nm, b in zip(self.NAMES, self.BITS)
                          for s in self.samples if s[2] & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def make_workload(torch, dims, seed):
    """Low-tubal-rank tensor (t-product of Gaussian factors, unit RMS) + outliers.

    Returned as the package's column-major flat CUDA buffer.  Data generation is
    setup (torch), outside every timed region.
    """
    n1, n2, n3 = dims
    r = WORKLOAD["tubal_rank"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((n3, r, n1), generator=g, device="cuda", dtype=torch.float32)
    b = torch.randn((n3, n2, r), generator=g, device="cuda", dtype=torch.float32)
    fx = torch.einsum("fjk,fki->fji", torch.fft.rfft(b, dim=0), torch.fft.rfft(a, dim=0))
    x = torch.fft.irfft(fx, n=n3, dim=0)  # (n3, n2, n1): column-major for (n1, n2, n3)
    x = x / x.pow(2).mean().sqrt()
    flat = x.reshape(-1).contiguous()
    k = int(round(WORKLOAD["outlier_frac"] * flat.numel()))
    idx = torch.randperm(flat.numel(), generator=g, device="cuda")[:k]
    flat[idx] = torch.rand(k, generator=g, device="cuda") * 2 - 1
    return flat


def lrta_bytes(shape, esize):
    """Algorithmic HBM bytes per randomized t-SVT by kernel category."""
    n1, n2, nf = shape[0], shape[1], math.prod(shape[2:])
    r0, r1 = WORKLOAD["ranks"]
    b0, b1 = WORKLOAD["blocks"]
    q0, q1 = WORKLOAD["krylov"]
    s0, s1 = (q0 + 1) * b0, (q1 + 1) * b1
    a0 = n1 * n2 * nf * esize          # mode-0 unfolding = the tensor
    a1 = n2 * r0 * nf * esize          # mode-1 unfolding of the mode-0 core
    return {
        "panel_sketch": a0 + a1,
        "panel_gram": q0 * a0 + q1 * a1,
        "proj_tc": a0 + a1 + (n2 * nf * s0 + r0 * nf * s1) * esize,   # read A, write W
        "gemm_expand": a0 + r0 * n2 * nf * esize,                      # write X, read C1
    }


def admm_bytes(shape, esize, nmodes=3):
    """Algorithmic HBM bytes per ADMM sweep of the non-LRTA kernels."""
    N = math.prod(shape)
    T = N * esize
    d = len(shape)
    # half spectrum along axis 0: (n0/2 + 1) / n0 of the complex volume
    S = 2 * esize * (shape[0] // 2 + 1) * (N // shape[0])
    # R2C (T in, S out), (d-2) forward + 1 solve + (d-2) inverse C2C passes, C2R (S in, T out)
    fft = (T + S) + (d - 2) * 2 * S + 2 * S + (d - 2) * 2 * S + (S + T)
    return {
        "fft": fft,
        # first sweep of a solve only (later sweeps get rhs from the fused tail)
        "admm_rhs": (3 + 2 * nmodes) * T + T,
        # L once + nmodes multipliers in, nmodes LRTA inputs out
        "lrta_input": (1 + 2 * nmodes) * T,
        # fused tail: L, L_prev, A, E, Y, mask + (G_new, G_old, lag) per mode in;
        # lag' per mode, E', Y', next rhs out
        "sweep_tail": (5 + 3 * nmodes) * T + N + (3 + nmodes) * T,
        # unfused fallbacks
        "lag_update": nmodes * 5 * T,
        "noise_dual": 6 * T + 2 * T + N,
    }


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200 import _lib
    from paper_2506_09594_b200.sketch import _run_lrta
    from paper_2506_09594_b200.solvers import NativeSolver
    from paper_2506_09594_b200.tensors import ColMajor

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    sharded = args.step == "tsvt-sharded"
    # under torchrun (any world size, 1 included) the rendezvous comes from its
    # environment: an explicit tcp:// store would wait for the agent's store
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif sharded:  # a one-rank NCCL group for the same code path
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=torch.device("cuda", local))
    lib = _lib.lib()
    dims = WORKLOAD["dims"]
    N = math.prod(dims)
    # replicas: a problem per rank; sharded: the same tensor on every rank
    flat = make_workload(torch, dims, 1234 if sharded else 1234 + rank)
    cm = ColMajor(flat, dims, "torch", None)
    if args.lrta == "blbp":
        sk = pk.SketchConfig(mode="fixed-accuracy", eps=BLBP_EPS, block=BLBP_BLOCK, seed=7)
    else:
        sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=WORKLOAD["ranks"],
                             blocks=WORKLOAD["blocks"], krylov=WORKLOAD["krylov"], seed=7)
    cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                          max_iters=max(1, args.steps))
    lam = cfg.lam_for(dims)
    mask_dev = torch.ones(N, dtype=torch.uint8, device="cuda")

    if args.step == "admm":
        run = NativeSolver("gnrhtc", cm, None, mask_dev, cfg, WORKLOAD["modes"], lam)
        stream = torch.cuda.ExternalStream(lib.tr_admm_stream(run.handle))
        lrta_per_step = len(WORKLOAD["modes"])

        def step():
            run.step()
    elif sharded:
        off, cnt = pk.shard_range(dims[-1], world, rank)
        face = dims[0] * dims[1]
        ldims = (dims[0], dims[1], cnt)
        cm_l = ColMajor(flat[face * off:face * (off + cnt)], ldims, "torch", None)
        tau = 0.05 * float(flat.norm()) / math.sqrt(N)
        stream = torch.cuda.current_stream()
        lrta_per_step = 1.0 / world  # every rank's step is 1/world of one t-SVT
        red = pk.DeviceAllreduce()

        def step():
            pk.gnhtsvt_randomized_sharded(cm_l, dims[-1], off, pk.Transform.fft(), pk.MCP(2.5),
                                          tau, sk, allreduce=red)
    else:
        out = ColMajor(torch.empty_like(flat), dims, "torch", None)
        tau = 0.05 * float(flat.norm()) / math.sqrt(N)
        stream = torch.cuda.current_stream()
        lrta_per_step = 1

        def step():
            _run_lrta(cm, out, WORKLOAD["ranks"], WORKLOAD["blocks"], WORKLOAD["krylov"], 7,
                      pk.Transform.fft(), pk.MCP(2.5), tau)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = lib.tr_launch_count()
    # timed region: no per-launch profiling events (they are taken afterwards,
    # in a separate untimed pass of the same steps)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.tr_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    prof_steps = max(1, min(args.steps, 5))
    lib.tr_profile_enable(1)
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    lib.tr_profile_enable(0)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = lrta_per_step * N * args.steps * world / (ms / 1e3)
    if args.step == "admm":
        run.close()

    # end to end through the public API with host (numpy) buffers: H2D of the
    # observations and mask, the sweeps, D2H of L and E, all inside the timer
    host = flat.reshape(tuple(reversed(dims))).permute(2, 1, 0).cpu().numpy()
    host_mask = np.ones(dims, dtype=bool)
    e2e_iters = max(10, args.steps)
    if sharded:
        tf = pk.Transform.fft()
        host_l = np.ascontiguousarray(host[..., off:off + cnt])
        pk.gnhtsvt_randomized_sharded(host_l, dims[-1], off, tf, pk.MCP(2.5), tau, sk,
                                      allreduce=red)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_iters):
            res = pk.gnhtsvt_randomized_sharded(host_l, dims[-1], off, tf, pk.MCP(2.5), tau, sk,
                                                allreduce=red)
        e2e_s = (time.perf_counter() - t0) / e2e_iters
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": host_l.nbytes,
               "d2h_bytes_per_step": res.nbytes,
               "api": "paper_2506_09594_b200.gnhtsvt_randomized_sharded(numpy slice)",
               "per_rank_bytes": True}
    elif args.step == "admm":
        cfg_e2e = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                                  max_iters=e2e_iters, tol=1e-30)
        # untimed warm-up call: page-locked staging blocks and the solver's
        # memory pool are set up once per process, as in any serving loop
        warm = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                               max_iters=1, tol=1e-30)
        warm_out = pk.gnrhtc(host, host_mask, warm)
        del warm_out
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        l_h, e_h, rep = pk.gnrhtc(host, host_mask, cfg_e2e)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": lrta_per_step * N * rep.iterations / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": (host.nbytes + host_mask.nbytes) / rep.iterations,
               "d2h_bytes_per_step": (l_h.nbytes + e_h.nbytes) / rep.iterations,
               "api": f"paper_2506_09594_b200.gnrhtc(numpy, max_iters={rep.iterations})",
               "admm_iters_per_s": rep.iterations / e2e_s}
    else:
        tf = pk.Transform.fft()
        tau = 0.05 * float(flat.norm()) / math.sqrt(N)
        pk.gnhtsvt_randomized(host, tf, pk.MCP(2.5), tau, sk)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_iters):
            res = pk.gnhtsvt_randomized(host, tf, pk.MCP(2.5), tau, sk)
        e2e_s = (time.perf_counter() - t0) / e2e_iters
        e2e = {"value": N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": host.nbytes,
               "d2h_bytes_per_step": res.nbytes,
               "api": "paper_2506_09594_b200.gnhtsvt_randomized(numpy)"}

    # roofline of the dominant HBM-bound kernel category
    peak, peak_kind = peaks()
    algo = {k: v * lrta_per_step for k, v in lrta_bytes(dims, 4).items()}
    if args.step == "admm":
        algo.update(admm_bytes(dims, 4, len(WORKLOAD["modes"])))
    # The north_star's named target, the batched Krylov products, measured on
    # their own: a standalone t-SVT of the same resident tensor (one stream,
    # nothing concurrent), panel passes timed by events on their stream.
    roof_k = None
    prof_k, reps_k = None, 1
    if rank == 0 and not sharded:
        out_k = ColMajor(torch.empty_like(flat), dims, "torch", None)
        tau_k = 0.05 * float(flat.norm()) / math.sqrt(N)

        def tsvt():
            _run_lrta(cm, out_k, WORKLOAD["ranks"], WORKLOAD["blocks"], WORKLOAD["krylov"], 7,
                      pk.Transform.fft(), pk.MCP(2.5), tau_k)
        tsvt()
        torch.cuda.synchronize()
        lib.tr_profile_enable(1)
        reps = reps_k = 3
        for _ in range(reps):
            tsvt()
        torch.cuda.synchronize()
        prof_k = _lib.profile_read()
        lib.tr_profile_enable(0)
        algo_k = lrta_bytes(dims, 4)
        roof_k = {}
        for cat in ("panel_gram", "panel_sketch"):
            if cat in prof_k:
                ms_k = prof_k[cat][0] / reps
                ach = algo_k[cat] / (ms_k / 1e3) / 1e9
                roof_k[cat] = {"achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                               "frac": round(ach / peak, 4), "ms_per_tsvt": round(ms_k, 4),
                               "launches_per_tsvt": prof_k[cat][1] / reps,
                               "algorithmic_bytes_per_tsvt": algo_k[cat]}
        roof_k["how"] = ("standalone randomized t-SVT of the bench tensor (no concurrent streams); "
                         "includes the small mode-1 passes")
        del out_k
    # Dominant kernel category by UNCONTENDED device time per step.  The per-mode
    # t-SVT chains of an ADMM sweep run on concurrent streams, so the event times
    # of their kernels overlap one another (a pass that queues behind another
    # mode's pass is charged the wait); for those categories the time comes from
    # the standalone t-SVT above (x t-SVTs per step).  The main-stream kernels of
    # the sweep (FFT solve, t-SVT inputs, fused tail) run with nothing beside them.
    cats = {k: v[0] / prof_steps for k, v in prof.items() if k in algo}
    src = {k: "sweep pass (main stream, nothing concurrent)" for k in cats}
    nl = {k: prof[k][1] / prof_steps for k in cats}
    if args.step == "admm" and prof_k is not None:
        for k in cats:
            if k in prof_k:
                cats[k] = prof_k[k][0] / reps_k * lrta_per_step
                nl[k] = prof_k[k][1] / reps_k * lrta_per_step
                src[k] = "standalone t-SVT pass (one stream) x t-SVTs per step"
    dom = max(cats, key=lambda k: cats[k]) if cats else None
    roof = None
    if dom:
        per_step_ms = cats[dom]
        achieved = algo[dom] / (per_step_ms / 1e3) / 1e9
        tcat, tsrc = measured_traffic()
        traffic = tcat.get(dom, {}).get("bytes_per_step")
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_unit": "DRAM bytes per step (ncu, summed over launches)",
                "traffic_source": tsrc, "share_of_step": round(per_step_ms / ms_per_step, 4),
                "algorithmic_bytes_per_step": algo[dom],
                "launches_per_step": nl[dom], "kernel_ms_per_step": round(per_step_ms, 4),
                "timed_in": src[dom],
                "note": "kernel time from CUDA events on the kernel's own stream in a separate "
                        "untimed pass; the dominant category is chosen by uncontended time "
                        "(kernel_ms_per_step below holds the raw event times of the concurrent "
                        "sweep, where the three mode streams overlap)"}
    extra = {}
    if rank == 0 and args.step == "admm" and not args.no_legs:
        extra["fp64"] = fp64_leg(torch, pk, NativeSolver, ColMajor, lib, flat, dims, mask_dev,
                                 min(args.steps, 10))
        extra["blbp"] = blbp_leg(torch, pk, ColMajor, lib, cm, dims)
    breakdown = {k: round(v[0] / prof_steps, 4)
                 for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian-factor t-product + uniform outliers)",
            "config": {"workload": WORKLOAD["workload"], "step": args.step, "dims": list(dims),
                       "ranks": list(WORKLOAD["ranks"]), "blocks": list(WORKLOAD["blocks"]),
                       "krylov": list(WORKLOAD["krylov"]), "gradient_modes": list(WORKLOAD["modes"]),
                       "parallelism": (f"last-mode-shard{world}" if sharded
                                       else f"replicas{world}"),
                       "l2": "every tensor 512 MB > 126 MB L2 (no flush needed)"},
            "admm_iters_per_s": (1e3 / ms_per_step) if args.step == "admm" else None,
            "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "roofline_krylov": roof_k,
            "kernel_ms_per_step": breakdown, "clocks": clk.summary(),
        }
        line["config"]["lrta"] = ("block Krylov (fixed-rank BKI: ranks 25, b 7, q 3) -- BASELINE "
                                  "configs[1] names block Lanczos bidiagonalisation; its "
                                  "fixed-accuracy leg is the 'blbp' object" if args.lrta == "bki"
                                  else f"block Lanczos bidiagonalisation (fixed-accuracy, "
                                       f"eps {BLBP_EPS}, block {BLBP_BLOCK})")
        line.update(extra)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.step, full=args.step == "admm")
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


BLBP_EPS, BLBP_BLOCK = 0.45, 8


def fp64_leg(torch, pk, NativeSolver, ColMajor, lib, flat, dims, mask_dev, steps):
    """The same ADMM sweep at the reference's precision (fp64 streams), timed
    with CUDA events on the solver's stream (3 warm-up sweeps)."""
    N = math.prod(dims)
    cm64 = ColMajor(flat.double(), dims, "torch", None)
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=WORKLOAD["ranks"],
                         blocks=WORKLOAD["blocks"], krylov=WORKLOAD["krylov"], seed=7)
    cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                          max_iters=steps + 3)
    run = NativeSolver("gnrhtc", cm64, None, mask_dev, cfg, WORKLOAD["modes"],
                       cfg.lam_for(dims))
    st = torch.cuda.ExternalStream(lib.tr_admm_stream(run.handle))
    for _ in range(3):
        run.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        run.step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    run.close()
    del cm64
    torch.cuda.empty_cache()
    return {"dtype": "f64", "value": len(WORKLOAD["modes"]) * N / (ms / 1e3), "unit": UNIT,
            "ms_per_step": ms, "steps": steps, "warmup": 3,
            "how": "same workload and sweep, fp64 tensors (the reference's precision), CUDA "
                   "events on the solver stream"}


def blbp_leg(torch, pk, ColMajor, lib, cm, dims, reps=3):
    """One fixed-accuracy (block Lanczos, sketch.py:287-403) randomized t-SVT of
    the bench tensor through the public API, device-resident input."""
    N = math.prod(dims)
    sk = pk.SketchConfig(mode="fixed-accuracy", eps=BLBP_EPS, block=BLBP_BLOCK, seed=7)
    tau = 0.05 * float(cm.flat.norm()) / math.sqrt(N)
    pk.gnhtsvt_randomized(cm, pk.Transform.fft(), pk.MCP(2.5), tau, sk)
    torch.cuda.synchronize()
    launches0 = lib.tr_launch_count()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = pk.gnhtsvt_randomized(cm, pk.Transform.fft(), pk.MCP(2.5), tau, sk)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    launches = (lib.tr_launch_count() - launches0) / reps
    del out
    _, diag = pk.ad_rsthosvd_blbp(cm, BLBP_EPS, block=BLBP_BLOCK, order=(0, 1), seed=7)
    torch.cuda.empty_cache()
    return {"value": N / dt, "unit": UNIT, "ms_per_tsvt": dt * 1e3, "eps": BLBP_EPS,
            "block": BLBP_BLOCK, "ranks": [diag.ranks[0], diag.ranks[1]],
            "iterations": [diag.iterations[0], diag.iterations[1]],
            "deflations": [diag.deflations[0], diag.deflations[1]],
            "launches_per_tsvt": launches,
            "how": "wall clock of the host-driven call (two small D2H per bidiagonalisation "
                   "step), device-resident input"}


def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def _slab(nf, seed):
    import numpy as np
    n1, n2, _ = WORKLOAD["dims"]
    rng = np.random.default_rng(seed)
    r = WORKLOAD["tubal_rank"]
    a = np.fft.rfft(rng.standard_normal((n1, r, nf)), axis=2)
    b = np.fft.rfft(rng.standard_normal((r, n2, nf)), axis=2)
    x = np.fft.irfft(np.einsum("ikf,kjf->ijf", a, b), n=nf, axis=2)
    x /= np.sqrt(np.mean(x ** 2))
    flat = x.ravel()
    k = int(round(WORKLOAD["outlier_frac"] * flat.size))
    idx = rng.choice(flat.size, size=k, replace=False)
    flat[idx] = rng.uniform(-1, 1, size=k)
    return flat.reshape(x.shape)


def _tenrec():
    """The unmodified reference package, installed once into baseline/_ref
    ("Reference arm"); None when it is absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "tenrec")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import tenrec
        return tenrec
    except Exception:
        return None


def tenrec_sweeps(tenrec, x, iters=1):
    """Seconds of ``iters`` GNRHTC sweeps of the reference itself: the loop body
    of tenrec/solvers.py:226-268 composed from tenrec's public functions
    (solve_grad_system, grad, gnhtsvt_randomized with the bench sketch, gnhtt,
    kkt_diagnostics) in the reference's order.  The end-of-solve objective
    (full face SVDs, solvers.py:274-282) is per solve, not per sweep, and is
    not timed."""
    import numpy as np

    dims = x.shape
    modes = WORKLOAD["modes"]
    sk = tenrec.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=WORKLOAD["ranks"],
                             blocks=WORKLOAD["blocks"], krylov=WORKLOAD["krylov"], seed=7)
    cfg = tenrec.SolverConfig(phi=tenrec.MCP(2.5), psi=tenrec.MCP(2.5), randomized=True,
                              sketch=sk, tol=1e-30, max_iters=iters)
    gset = tenrec.GradientSet(dims, modes)
    lam = cfg.lam_for(dims)
    gamma = len(modes)
    maskf = np.ones(dims)
    zeros = lambda: np.zeros(dims)  # noqa: E731
    l, e, y = zeros(), zeros(), zeros()
    g = {k: zeros() for k in modes}
    lag = {k: zeros() for k in modes}
    mu = cfg.mu0
    t0 = time.perf_counter()
    for _ in range(iters):
        b = x - e + y / mu
        l_new = tenrec.solve_grad_system(b, {k: g[k] - lag[k] / mu for k in modes}, gset)
        tau = 1.0 / (gamma * mu)
        grad_l = {k: tenrec.grad(l_new, k) for k in modes}
        g_new = {k: tenrec.gnhtsvt_randomized(grad_l[k] + lag[k] / mu, cfg.transform, cfg.phi,
                                              tau, cfg.sketch) for k in modes}
        h = x - l_new + y / mu
        e_new = maskf * tenrec.gnhtt(maskf * h, cfg.psi, lam / mu, cfg.structure) \
            + (1.0 - maskf) * h
        y = y + mu * (x - l_new - e_new)
        for k in modes:
            lag[k] = lag[k] + mu * (grad_l[k] - g_new[k])
        tenrec.kkt_diagnostics(tenrec.SolverState(m=x, l=l_new, e=e_new, g=g_new, grad_l=grad_l,
                                                  l_prev=l, e_prev=e, g_prev=g))
        l, e, g = l_new, e_new, g_new
        mu = min(cfg.mu_max, cfg.growth * mu)
    return time.perf_counter() - t0


def _full_config_x():
    """The bench tensor itself (bench.make_workload, seed 1234) as fp64 numpy,
    generated on the GPU when one is visible, else the slab generator."""
    import numpy as np

    try:
        import torch

        if torch.cuda.is_available():
            dims = WORKLOAD["dims"]
            flat = make_workload(torch, dims, 1234)
            x = flat.reshape(tuple(reversed(dims))).permute(2, 1, 0).cpu().numpy()
            del flat
            torch.cuda.empty_cache()
            return np.asfortranarray(x, dtype=np.float64)
    except Exception:
        pass
    return _slab(WORKLOAD["dims"][2], 1234)


def cpu_baseline(step="admm", nf=8, seed=0, iters=1, full=False):
    """The reference timed on the host cores on a bounded sample: ``iters``
    GNRHTC sweeps (or one t-SVT) of a 1024x1024x``nf`` slab.  tenrec itself
    (baseline/_ref, kind "reference") when installed, else the oracle port.
    ``full``: one sweep of the whole 1024x1024x128 bench tensor beside it, which
    checks the per-voxel extrapolation from the slab."""
    import numpy as np

    from oracle import admm, lrta, philox
    from oracle.tensor_ops import TransformSpec

    tenrec = _tenrec()
    x = _slab(nf, seed)
    spec = TransformSpec("fft")
    mcp = (2, 2.5, 0.0)

    def thr(a, tau):
        return lrta.gnhtsvt_randomized(a, spec, mcp, tau, WORKLOAD["ranks"], WORKLOAD["blocks"],
                                       WORKLOAD["krylov"], (0, 1), philox.PhiloxSketchSource(7))

    kind = "reference" if tenrec is not None else "port"
    who = "tenrec 0.1.0 (baseline/_ref)" if tenrec is not None else "fp64 numpy oracle port"
    if step == "admm":
        if tenrec is not None:
            dt = tenrec_sweeps(tenrec, x, iters)
        else:
            t0 = time.perf_counter()
            admm.admm_complete(x, np.ones(x.shape, dtype=bool), thr, mcp,
                               admm.default_lambda(x.shape), WORKLOAD["modes"], max_iters=iters,
                               tol=1e-30)
            dt = time.perf_counter() - t0
        vox = len(WORKLOAD["modes"]) * x.size * iters
        sample = f"{iters} GNRHTC sweep(s) of a 1024x1024x{nf} slab ({who}, fp64)"
    else:
        t0 = time.perf_counter()
        if tenrec is not None:
            sk = tenrec.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=WORKLOAD["ranks"],
                                     blocks=WORKLOAD["blocks"], krylov=WORKLOAD["krylov"], seed=7)
            tenrec.gnhtsvt_randomized(x, tenrec.Transform.fft(), tenrec.MCP(2.5), 0.05, sk)
        else:
            thr(x, 0.05)
        dt = time.perf_counter() - t0
        vox = x.size
        sample = f"one randomized t-SVT of a 1024x1024x{nf} slab ({who}, fp64)"
    out = {"value": vox / dt, "unit": UNIT, "cores": _threads(), "kind": kind,
           "sample": sample, "seconds": dt}
    if full and step == "admm" and tenrec is not None:
        xf = _full_config_x()
        dtf = tenrec_sweeps(tenrec, xf, 1)
        out["full_config"] = {
            "value": len(WORKLOAD["modes"]) * xf.size / dtf, "unit": UNIT, "seconds": dtf,
            "sample": "1 GNRHTC sweep of the whole 1024x1024x128 bench tensor (tenrec, fp64)",
            "slab_extrapolation_ratio": (vox / dt) / (len(WORKLOAD["modes"]) * xf.size / dtf)}
        del xf
    return out


def run_reference(args):
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    nf = 4
    for w in range(args.warmup):
        cpu_baseline(args.step, nf=nf, seed=100 + w)
    vals, secs = [], 0.0
    for s in range(args.steps):
        r = cpu_baseline(args.step, nf=nf, seed=s)
        vals.append(r["value"])
        secs += r["seconds"]
    value = statistics.mean(vals)
    sample = r["sample"]
    full = cpu_baseline(args.step, nf=nf, seed=0, full=True).get("full_config") \
        if not args.no_cpu_baseline else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Gaussian-factor t-product + uniform outliers)",
        "impl": "reference",
        "config": {"workload": WORKLOAD["workload"], "step": args.step,
                   "sample": "per step: " + sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _threads(), "kind": r["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if full:
        line["full_config"] = full
    print(json.dumps(line), flush=True)


CONFIGS = {
    2: {"workload": "completion-512x512x16x32-f32", "dims": (512, 512, 16, 32),
        "tubal_rank": 15, "noise": 0.01, "observed": 0.10, "ranks": (25, 25), "blocks": (9, 9),
        "krylov": (2, 2), "solver": "gnhtc",
        "note": "BASELINE configs[2]: order-4 completion, transform along modes 3 and 4, q = 2, "
                "p = 10 (target rank 15 + 10)"},
    3: {"workload": "onebit-2048x2048x64-f32", "dims": (2048, 2048, 64), "tubal_rank": 10,
        "observed": 0.50, "ranks": (15, 15), "blocks": (5, 5), "krylov": (2, 2),
        "solver": "gnobhtc", "theta": 1.5, "sigma": 0.1,
        "note": "BASELINE configs[3]: one-bit recovery, 50% sampled, q = 2, p = 5 (target rank "
                "10 + 5); dithered signs (theta 1.5, Gaussian noise 0.1) as in tenrec.onebit"},
}


def make_tproduct(torch, dims, r, seed):
    """Gaussian factors n1 x r x trailing and r x n2 x trailing, t-product along
    every trailing mode (FFT over the trailing axes), unit RMS; column-major flat."""
    n1, n2 = dims[0], dims[1]
    tr = tuple(dims[2:])
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(tr[::-1] + (r, n1), generator=g, device="cuda")  # (..., k, i)
    b = torch.randn(tr[::-1] + (n2, r), generator=g, device="cuda")  # (..., j, k)
    ax = tuple(range(len(tr)))
    fa, fb = torch.fft.fftn(a, dim=ax), torch.fft.fftn(b, dim=ax)
    x = torch.fft.ifftn(torch.matmul(fb, fa), dim=ax).real  # (..., j, i): column-major
    x = x / x.pow(2).mean().sqrt()
    return x.reshape(-1).contiguous(), g


def run_config(args):
    """One ADMM sweep of BASELINE configs[2] or configs[3] (N = 1; same line
    contract as the default step; e2e through gnhtc / gnobhtc with host arrays)."""
    import numpy as np
    import torch

    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200 import _lib
    from paper_2506_09594_b200.solvers import NativeSolver
    from paper_2506_09594_b200.tensors import ColMajor

    C = CONFIGS[args.config]
    torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
    lib = _lib.lib()
    dims = C["dims"]
    N = math.prod(dims)
    modes = tuple(range(len(dims)))
    x, g = make_tproduct(torch, dims, C["tubal_rank"], 4242)
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=C["ranks"], blocks=C["blocks"],
                         krylov=C["krylov"], seed=7)
    if C["solver"] == "gnhtc":
        x = x + C["noise"] * torch.randn(N, generator=g, device="cuda")
        mask = torch.rand(N, generator=g, device="cuda") < C["observed"]
        mobs = torch.where(mask, x, torch.zeros_like(x))
        cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                              max_iters=args.steps + args.warmup, tol=1e-30)
        cm = ColMajor(mobs, dims, "torch", None)
        run = NativeSolver("gnhtc", cm, None, mask.to(torch.uint8), cfg, modes,
                           cfg.lam_for(dims))
        host_in = (mobs.reshape(dims[::-1]).permute(*reversed(range(len(dims)))).cpu().numpy(),
                   mask.reshape(dims[::-1]).permute(*reversed(range(len(dims)))).cpu().numpy())
    else:
        x = x / x.abs().max()
        m = int(C["observed"] * N)
        idx = torch.randint(0, N, (m,), generator=g, device="cuda")
        y = x[idx] + C["sigma"] * torch.randn(m, generator=g, device="cuda")
        dither = (torch.rand(m, generator=g, device="cuda") * 2 - 1) * C["theta"]
        sgn = torch.where(y + dither >= 0, 1.0, -1.0)
        j2 = torch.bincount(idx, minlength=N).float()
        j1 = C["theta"] * torch.bincount(idx, weights=sgn, minlength=N).float()
        cfg = pk.SolverConfig.one_bit(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True,
                                      sketch=sk, max_iters=args.steps + args.warmup, tol=1e-30)
        run = NativeSolver("gnobhtc", ColMajor(j1, dims, "torch", None),
                           ColMajor(j2, dims, "torch", None), None, cfg, modes,
                           cfg.lam_for(dims), alpha=1.0, mcount=float(m))
        host_in = (idx.cpu().numpy(), sgn.to(torch.int8).cpu().numpy(), j1, j2, m)
    stream = torch.cuda.ExternalStream(lib.tr_admm_stream(run.handle))
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.tr_launch_count()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            run.step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.tr_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    lib.tr_profile_enable(1)
    for _ in range(2):
        run.step()
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    lib.tr_profile_enable(0)
    run.close()
    value = len(modes) * N / (ms / 1e3)
    # end to end through the public API with host arrays
    e2e_iters = 3
    if C["solver"] == "gnhtc":
        mo_h, mk_h = host_in
        cfg_e = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                                max_iters=e2e_iters, tol=1e-30)
        t0 = time.perf_counter()
        l_h, rep = pk.gnhtc(mo_h, mk_h, cfg_e)
        e2e_s = time.perf_counter() - t0
        h2d, d2h = mo_h.nbytes + mk_h.nbytes, l_h.nbytes
        api = f"paper_2506_09594_b200.gnhtc(numpy, max_iters={e2e_iters})"
    else:
        idx_h, sgn_h, j1, j2, m = host_in
        dims_f = tuple(dims)
        perm = tuple(reversed(range(len(dims))))
        obs = pk.ObservationSet(dims=dims_f, theta=C["theta"], indices=idx_h, signs=sgn_h,
                                j1=j1.reshape(dims[::-1]).permute(*perm).cpu().numpy(),
                                j2=j2.reshape(dims[::-1]).permute(*perm).cpu().numpy())
        cfg_e = pk.SolverConfig.one_bit(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True,
                                        sketch=sk, max_iters=e2e_iters, tol=1e-30)
        t0 = time.perf_counter()
        l_h, rep = pk.gnobhtc(obs, cfg_e, alpha=1.0)
        e2e_s = time.perf_counter() - t0
        h2d, d2h = obs.j1.nbytes + obs.j2.nbytes, np.asarray(l_h).nbytes
        api = f"paper_2506_09594_b200.gnobhtc(ObservationSet f32, max_iters={e2e_iters})"
    # roofline: the dominant HBM category with its algorithmic bytes
    peak, peak_kind = peaks()
    algo = admm_bytes(dims, 4, len(modes))
    cats = {k: v for k, v in prof.items() if k in algo and k != "admm_rhs"}
    dom = max(cats, key=lambda k: cats[k][0]) if cats else None
    roof = None
    if dom:
        per_ms = cats[dom][0] / 2
        ach = algo[dom] / (per_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": None, "algorithmic_bytes_per_step": algo[dom],
                "share_of_step": round(per_ms / ms, 4)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Gaussian-factor t-product)",
        "config": {"workload": C["workload"], "step": "admm", "dims": list(dims),
                   "ranks": list(C["ranks"]), "blocks": list(C["blocks"]),
                   "krylov": list(C["krylov"]), "gradient_modes": list(modes),
                   "solver": C["solver"], "parallelism": "replicas1", "note": C["note"]},
        "admm_iters_per_s": 1e3 / ms,
        "e2e": {"value": len(modes) * N * rep.iterations / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": h2d / rep.iterations, "d2h_bytes_per_step": d2h / rep.iterations,
                "api": api},
        "gpu_launches": launches, "roofline": roof,
        "kernel_ms_per_step": {k: round(v[0] / 2, 4)
                               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


CONFIG4 = {
    "workload": "robust-completion-2048x2048x32x(4N)-f32",
    "local_dims": (2048, 2048, 32, 4),
    "tubal_rank": 30,
    "observed": 0.20,
    "outlier_frac": 0.05,
    "outlier_amp": 5.0,
    "ranks": (40, 40),
    "blocks": (10, 10),
    "krylov": (3, 3),
}


def make_config4_slab(torch, world, rank, seed=4321):
    """This rank's slab of BASELINE configs[4]'s tensor at world size N: global
    dims (2048, 2048, 32, 4N) -- exactly configs[4] at N = 8 -- as
    sum_{r<30} a_r(i0) b_r(i1) c_r(i2, i3) with Gaussian factors (tubal rank <= 30),
    unit RMS, 5% outliers U[-5, 5], 20% observed.  Every rank draws the shared
    factors from the same seed and slices c along the last mode, so the slabs
    tile one global tensor.  Setup only (outside every timed region)."""
    n0, n1, n2, nl = CONFIG4["local_dims"]
    r = CONFIG4["tubal_rank"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((n0, r), generator=g, device="cuda")
    b = torch.randn((n1, r), generator=g, device="cuda")
    c = torch.randn((n2, nl * world, r), generator=g, device="cuda")[:, rank * nl:(rank + 1) * nl]
    # column-major flat (i0 fastest): x[i3, i2, i1, i0] in C order
    x = torch.einsum("ir,jr,klr->lkji", a, b, c).contiguous() / math.sqrt(r)
    flat = x.reshape(-1)
    gl = torch.Generator(device="cuda").manual_seed(seed + 1 + rank)
    out = torch.rand(flat.numel(), generator=gl, device="cuda") < CONFIG4["outlier_frac"]
    amp = CONFIG4["outlier_amp"]
    flat = torch.where(out, (torch.rand(flat.numel(), generator=gl, device="cuda") * 2 - 1) * amp,
                       flat)
    mask = (torch.rand(flat.numel(), generator=gl, device="cuda") < CONFIG4["observed"])
    flat = torch.where(mask, flat, torch.zeros_like(flat))
    return flat.contiguous(), mask.to(torch.uint8)


def run_admm_sharded(args):
    """One GNRHTC sweep of configs[4] sharded along the last mode over the N
    ranks (tr_admm_create_sharded; weak scaling, 4 faces per rank)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_09594_b200 as pk
    from paper_2506_09594_b200 import _lib
    from paper_2506_09594_b200.shard import DeviceComm, ShardedSolver
    from paper_2506_09594_b200.tensors import ColMajor

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # torchrun: its own rendezvous
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=torch.device("cuda", local))
    lib = _lib.lib()
    ldims = CONFIG4["local_dims"]
    gdims = ldims[:-1] + (ldims[-1] * world,)
    Nl = math.prod(ldims)
    flat, mask = make_config4_slab(torch, world, rank)
    cm = ColMajor(flat, ldims, "torch", None)
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=CONFIG4["ranks"],
                         blocks=CONFIG4["blocks"], krylov=CONFIG4["krylov"], seed=7)
    cfg = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                          max_iters=args.steps + args.warmup, tol=1e-30)
    comm = DeviceComm()
    modes = tuple(range(len(ldims)))
    run = ShardedSolver("gnrhtc", cm, mask, cfg, modes, cfg.lam_for(gdims), gdims[-1],
                        rank * ldims[-1], comm)
    stream = torch.cuda.ExternalStream(run.stream())
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.tr_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            run.step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.tr_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    run.close()
    ms_per_step = ms / args.steps
    value = len(modes) * Nl * world * args.steps / (ms / 1e3)
    # end to end through the public API, host slabs in / out
    host = flat.reshape(tuple(reversed(ldims))).permute(3, 2, 1, 0).cpu().numpy()
    host_mask = mask.reshape(tuple(reversed(ldims))).permute(3, 2, 1, 0).cpu().numpy().astype(bool)
    del flat, mask, cm
    torch.cuda.empty_cache()
    e2e_iters = 3
    cfg_e = pk.SolverConfig(phi=pk.MCP(2.5), psi=pk.MCP(2.5), randomized=True, sketch=sk,
                            max_iters=e2e_iters, tol=1e-30)
    dist.barrier()
    t0 = time.perf_counter()
    l_h, e_h, rep = pk.gnrhtc_sharded(host, host_mask, cfg_e, gdims[-1], rank * ldims[-1], comm)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian CP factors, tubal rank <= 30, 5% outliers "
                    "U[-5, 5], 20% observed)",
            "config": {"workload": CONFIG4["workload"], "step": "admm-sharded",
                       "global_dims": list(gdims), "local_dims": list(ldims),
                       "ranks": list(CONFIG4["ranks"]), "blocks": list(CONFIG4["blocks"]),
                       "krylov": list(CONFIG4["krylov"]), "gradient_modes": list(modes),
                       "parallelism": f"last-mode-shard{world}",
                       "note": "BASELINE configs[4] (2048x2048x32x32) at N = 8",
                       "l2": "every local tensor 2.1 GB > 126 MB L2 (no flush needed)"},
            "admm_iters_per_s": 1e3 / ms_per_step,
            "e2e": {"value": len(modes) * Nl * world * rep.iterations / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": (host.nbytes + host_mask.nbytes) / rep.iterations,
                    "d2h_bytes_per_step": (l_h.nbytes + e_h.nbytes) / rep.iterations,
                    "per_rank_bytes": True,
                    "api": f"paper_2506_09594_b200.gnrhtc_sharded(numpy slab, "
                           f"max_iters={rep.iterations})"},
            "gpu_launches": launches, "clocks": clk.summary(),
            "collective_calls": dict(comm.calls),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--step", choices=("admm", "lrta", "tsvt-sharded", "admm-sharded"),
                    default="admm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the fp64 and BLBP legs")
    ap.add_argument("--config", type=int, default=1, choices=(1, 2, 3),
                    help="BASELINE configs[k] of the ADMM step (1 = the bench default)")
    ap.add_argument("--lrta", choices=("bki", "blbp"), default="bki",
                    help="sketch of the ADMM step's t-SVTs: fixed-rank block Krylov (default) "
                         "or fixed-accuracy block Lanczos")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.step == "admm-sharded":
        run_admm_sharded(args)
    elif args.config in CONFIGS:
        run_config(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
