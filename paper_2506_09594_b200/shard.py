"""Multi-GPU randomized t-SVT and ADMM: one rank per GPU, the tensor sharded
along its last mode (row (e)).

For the reference algorithm -- Tucker compression of modes 0 and 1 by block
Krylov sketching, then the transform-domain SVT of the r0 x r1 x faces core
(tenrec/sketch.py:211-270, 430-456) -- a shard of the last mode is a block of
whole columns of both unfoldings.  Every rank therefore streams only its own
slice; what crosses ranks is small and fp64:

  * the n x b Krylov block of each power (sketch.py:253-259), summed over the
    column shards,
  * the s x s Ritz Gram W^T W (sketch.py:262-263),
  * the compressed core, which every rank then thresholds whole (the mode-3..N
    transform needs all faces) before expanding its own faces.

The sketch is drawn at GLOBAL column indices (counter-based Philox), so each
rank's output slice equals the same slice of the single-GPU result up to fp64
summation order.  The sums go through `tr_allreduce_fn`: in production an
in-place ``torch.distributed.all_reduce`` (NCCL over NVLink) ordered on the
t-SVT's stream, so no host synchronisation is added.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .penalties import encode as encode_penalty
from .sketch import SketchConfig, _resolve
from .tensors import ColMajor, empty_like, from_device, to_device, workspace
from .transform import DEFAULT_TRANSFORM, as_transform

__all__ = ["shard_range", "allreduce_tensor", "DeviceAllreduce", "gnhtsvt_randomized_sharded",
           "DeviceComm", "gnrhtc_sharded", "gnhtc_sharded"]


def shard_range(n: int, world: int, rank: int):
    """(offset, length) of rank's contiguous block of n items (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    base, extra = divmod(int(n), int(world))
    off = rank * base + min(rank, extra)
    return off, base + (1 if rank < extra else 0)


def allreduce_tensor(t, group=None):
    """In-place sum across the ranks of ``group`` (any torch.distributed backend)."""
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of device memory (fp64 or bytes)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "stream": None}


class DeviceAllreduce:
    """A ``tr_allreduce_fn`` backed by torch.distributed (NCCL on GPU boxes).

    The callback wraps the device buffer without copying and issues the
    all-reduce with the t-SVT's stream as torch's current stream, so NCCL waits
    for the kernels that produced the partials and the following kernels wait
    for NCCL -- stream order end to end.
    """

    def __init__(self, group=None):
        self.group = group
        self.calls = 0
        self.error = None
        self.fn = _lib.ALLREDUCE_FN(self._callback)

    def _callback(self, buf, count, stream, user):
        import torch

        try:
            ptr = ctypes.cast(buf, ctypes.c_void_p).value
            t = torch.as_tensor(_CudaArray(ptr, count), device="cuda")
            with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                allreduce_tensor(t, self.group)
            self.calls += 1
            return 0
        except Exception as exc:  # surfaced by the caller
            self.error = exc
            return 1


def gnhtsvt_randomized_sharded(a_local, last_all: int, last_off: int,
                               transform=DEFAULT_TRANSFORM, penalty=None, tau: float = 0.0,
                               sketch: SketchConfig = None, allreduce=None, group=None):
    """This rank's slice of ``gnhtsvt_randomized`` of the whole tensor.

    ``a_local`` holds indices ``[last_off, last_off + a_local.shape[-1])`` of
    the last mode (length ``last_all`` overall); every rank must call with the
    same transform / penalty / tau / sketch.  ``allreduce`` is a
    :class:`DeviceAllreduce` (default: one over ``group``).  Returns the output
    slice in ``a_local``'s container.
    """
    if sketch is None:
        raise ValueError("a sketch configuration is required")
    if penalty is None:
        raise ValueError("a penalty is required")
    if tau < 0:
        raise ValueError("tau must be >= 0")
    transform = as_transform(transform)
    cm = a_local if isinstance(a_local, ColMajor) else to_device(a_local)
    dims = cm.dims
    if len(dims) < 3:
        raise ValueError(f"tensor order {len(dims)} < required 3")
    if not (0 <= last_off and last_off + dims[-1] <= last_all):
        raise ValueError(f"shard [{last_off}, {last_off + dims[-1]}) outside [0, {last_all})")
    gdims = tuple(dims[:-1]) + (int(last_all),)
    transform.check_shape(gdims)
    sketch, ranks, blocks, krylov = _resolve(sketch, gdims)
    if allreduce is None:
        allreduce = DeviceAllreduce(group)
    lib = _lib.lib()
    rk, bl, kr = _lib.i64(ranks), _lib.i64(blocks), _lib.i64(krylov)
    nbytes = lib.tr_lrta_workspace(cm.dtype_code, len(gdims), _lib.i64(gdims), rk, bl, kr)
    if nbytes < 0:
        _lib.check(1)
    ws = workspace(nbytes)
    out = empty_like(cm)
    kind, p0, p1 = encode_penalty(penalty)
    tcode, tmats, talphas, keep_t = transform.device_args(gdims)
    rc = lib.tr_gnhtsvt_randomized_sharded(
        cm.dtype_code, ctypes.c_void_p(cm.ptr), ctypes.c_void_p(out.ptr), len(dims),
        _lib.i64(dims), int(last_all), int(last_off), rk, bl, kr,
        ctypes.c_uint64(int(sketch.seed) & (2 ** 64 - 1)), tcode, tmats, talphas, kind, p0, p1,
        float(tau), allreduce.fn, None, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
        _lib.stream_ptr())
    del keep_t
    if rc and getattr(allreduce, "error", None) is not None:
        raise _lib.CudaPathError(f"all-reduce failed: {allreduce.error!r}")
    _lib.check(rc)
    return out if isinstance(a_local, ColMajor) else from_device(out)


# -- the sharded ADMM (tr_admm_create_sharded) ---------------------------------

class DeviceComm:
    """The ``tr_comm`` collectives of the sharded ADMM over torch.distributed.

    ``staged=False`` (NCCL): the callbacks wrap the device buffers without a
    copy and issue the collective with the solver's stream as torch's current
    stream -- stream-ordered, NVLink all-to-all / peer sends.  ``staged=True``
    (any CPU backend, e.g. gloo; used to run several ranks on one test GPU):
    each callback synchronises the stream, stages the bytes through host
    memory, runs the collective there and copies the result back.
    """

    def __init__(self, group=None, staged=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.staged = (dist.get_backend(group) != "nccl") if staged is None else bool(staged)
        self.error = None
        self.calls = {"allreduce": 0, "alltoall": 0, "halo": 0}
        self._fns = (_lib.COMM_ALLREDUCE_FN(self._allreduce), _lib.COMM_ALLTOALL_FN(self._alltoall),
                     _lib.COMM_HALO_FN(self._halo))
        self.struct = _lib.TrComm(self.world, self.rank, self._fns[0], self._fns[1], self._fns[2],
                                  None)

    # device views ---------------------------------------------------------
    @staticmethod
    def _view(ptr, count, typestr):
        import torch

        return torch.as_tensor(_CudaArray(ptr, count, typestr), device="cuda")

    def _run(self, name, stream, body):
        import torch

        try:
            with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                body()
                if self.staged:
                    torch.cuda.current_stream().synchronize()
            self.calls[name] += 1
            return 0
        except Exception as exc:  # surfaced by the caller
            self.error = exc
            return 1

    def _allreduce(self, buf, count, op, stream, user):
        import torch.distributed as dist

        def body():
            t = self._view(ctypes.cast(buf, ctypes.c_void_p).value, count, "<f8")
            red = dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM
            if self.staged:
                h = t.cpu()
                dist.all_reduce(h, op=red, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=red, group=self.group)
        return self._run("allreduce", stream, body)

    def _alltoall(self, send, recv, nbytes, stream, user):
        import torch.distributed as dist

        def body():
            n = int(nbytes) * self.world
            s = self._view(send, n, "|u1")
            r = self._view(recv, n, "|u1")
            if self.staged:
                hs = s.cpu()
                hr = torch_empty_like_cpu(hs)
                if self.world == 1:
                    hr.copy_(hs)
                else:
                    dist.all_to_all_single(hr, hs, group=self.group)
                r.copy_(hr)
            else:
                dist.all_to_all_single(r, s, group=self.group)
        return self._run("alltoall", stream, body)

    def _halo(self, first, last, gprev, gnext, nbytes, stream, user):
        import torch.distributed as dist

        def body():
            n = int(nbytes)
            W, r = self.world, self.rank
            prev, nxt = (r - 1) % W, (r + 1) % W
            f, l_ = self._view(first, n, "|u1"), self._view(last, n, "|u1")
            gp, gn = self._view(gprev, n, "|u1"), self._view(gnext, n, "|u1")
            if self.staged:
                hf, hl = f.cpu(), l_.cpu()
                hp, hn = torch_empty_like_cpu(hf), torch_empty_like_cpu(hf)
                # my last face is the next rank's ghost_prev (tag 0), my first
                # face the previous rank's ghost_next (tag 1)
                reqs = [dist.isend(hl, _global(self.group, nxt), group=self.group, tag=0),
                        dist.isend(hf, _global(self.group, prev), group=self.group, tag=1),
                        dist.irecv(hp, _global(self.group, prev), group=self.group, tag=0),
                        dist.irecv(hn, _global(self.group, nxt), group=self.group, tag=1)]
                for q in reqs:
                    q.wait()
                gp.copy_(hp)
                gn.copy_(hn)
            else:
                # same issue order on every rank: with two ranks prev == next,
                # and NCCL pairs messages between two peers in issue order
                ops = [dist.P2POp(dist.isend, l_, _global(self.group, nxt), self.group),
                       dist.P2POp(dist.isend, f, _global(self.group, prev), self.group),
                       dist.P2POp(dist.irecv, gp, _global(self.group, prev), self.group),
                       dist.P2POp(dist.irecv, gn, _global(self.group, nxt), self.group)]
                for q in dist.batch_isend_irecv(ops):
                    q.wait()
        return self._run("halo", stream, body)


def torch_empty_like_cpu(t):
    import torch

    return torch.empty_like(t, device="cpu")


def _global(group, rank):
    import torch.distributed as dist

    return rank if group is None else dist.get_global_rank(group, rank)


class ShardedSolver:
    """One sharded GNRHTC / GNHTC run (tr_admm_create_sharded) on this rank's slab."""

    def __init__(self, kind, cm: ColMajor, mask_dev, cfg, modes, lam, last_all, last_off,
                 comm: DeviceComm):
        self.lib = _lib.lib()
        self.cm = cm
        self.comm = comm
        self.keep = [cm, mask_dev]
        dims = cm.dims
        gdims = tuple(dims[:-1]) + (int(last_all),)
        sk = cfg.sketch
        sk, ranks, blocks, krylov = _resolve(sk, gdims)
        phi = encode_penalty(cfg.phi)
        psi = encode_penalty(cfg.psi)
        handle = ctypes.c_void_p()
        rc = self.lib.tr_admm_create_sharded(
            cm.dtype_code, len(dims), _lib.i64(dims), 0 if kind == "gnrhtc" else 1,
            ctypes.c_void_p(cm.ptr), ctypes.c_void_p(mask_dev.data_ptr()), len(modes),
            _lib.i64(modes), phi[0], phi[1], phi[2], psi[0], psi[1], psi[2], float(lam),
            float(cfg.mu0), float(cfg.mu_max), float(cfg.growth), _lib.i64(ranks),
            _lib.i64(blocks), _lib.i64(krylov), ctypes.c_uint64(int(sk.seed) & (2 ** 64 - 1)),
            int(last_all), int(last_off), ctypes.byref(comm.struct), ctypes.byref(handle))
        self._check(rc)
        self.handle = handle
        self.out = (ctypes.c_double * 15)()

    def _check(self, rc):
        if rc and self.comm.error is not None:
            raise _lib.CudaPathError(f"collective failed: {self.comm.error!r}")
        _lib.check(rc)

    def step(self):
        self._check(self.lib.tr_admm_step(self.handle, self.out))
        return list(self.out)

    def read(self, which: int) -> ColMajor:
        import torch

        flat = torch.empty_like(self.cm.flat)
        _lib.check(self.lib.tr_admm_read(self.handle, which, ctypes.c_void_p(flat.data_ptr()),
                                         _lib.stream_ptr()))
        return ColMajor(flat, self.cm.dims, self.cm.kind, self.cm.np_dtype)

    def stream(self):
        return self.lib.tr_admm_stream(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.tr_admm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _sharded_complete(mobs_local, mask_local, cfg, last_all, last_off, comm, group, noise_free):
    import time

    import torch
    import torch.distributed as dist

    from .solvers import SolveReport
    from .tensors import mask_to_device

    t0 = time.perf_counter()
    cfg.validate()
    if not cfg.randomized:
        raise ValueError("the sharded solver needs randomized=True with a SketchConfig")
    if cfg.pure_lowrank:
        raise ValueError("the sharded solver runs the gradient chain (pure_lowrank=False)")
    if str(cfg.structure).lower() != "entry":
        raise ValueError("the sharded solver supports structure='entry'")
    comm = DeviceComm(group) if comm is None else comm
    cm = mobs_local if isinstance(mobs_local, ColMajor) else to_device(mobs_local)
    dims = cm.dims
    if tuple(mask_local.shape) != dims:
        raise ValueError("mask shape must match the observation tensor")
    mdev = mask_to_device(mask_local)
    gdims = tuple(dims[:-1]) + (int(last_all),)
    lam = cfg.lam_for(gdims)
    modes = cfg.device_modes(gdims)
    run = ShardedSolver("gnhtc" if noise_free else "gnrhtc", cm, mdev, cfg, modes, lam, last_all,
                        last_off, comm)
    report = SolveReport()
    try:
        for _ in range(cfg.max_iters):
            o = run.step()
            report.residual_history.append(o[0:5])
            report.diff_fro_history.append([o[5], o[6], o[7]])
            report.feas_fro_history.append([o[8], o[9]])
            report.multiplier_history.append([o[10], o[11]])
            report.mu_history.append(o[12])
            report.iterations += 1
            if max(o[0:5]) <= cfg.tol and max(o[5:8]) <= cfg.tol:
                report.converged = True
                break
        l_cm = run.read(0)
        e_cm = run.read(1)
    finally:
        run.close()
    fin = torch.tensor([float(torch.isfinite(l_cm.flat).all())], dtype=torch.float64)
    if comm.world > 1:
        dist.all_reduce(fin, op=dist.ReduceOp.MIN, group=group)
    if fin.item() < 1.0:
        raise FloatingPointError("solver produced non-finite iterates")
    report.objective = {"lambda": lam}
    report.wall_clock = time.perf_counter() - t0
    return from_device(l_cm), from_device(e_cm), report


def gnrhtc_sharded(mobs_local, mask_local, cfg, last_all: int, last_off: int, comm=None,
                   group=None):
    """Robust completion of a tensor sharded along its last mode over the ranks
    of ``group`` (one GPU each).  Every rank passes its slab of faces
    ``[last_off, last_off + mobs_local.shape[-1])``; the residual history is
    global.  Returns this rank's ``(L, E, report)`` slabs."""
    return _sharded_complete(mobs_local, mask_local, cfg, last_all, last_off, comm, group, False)


def gnhtc_sharded(mobs_local, mask_local, cfg, last_all: int, last_off: int, comm=None,
                  group=None):
    """Noise-free completion, sharded like :func:`gnrhtc_sharded`: ``(L, report)``."""
    l, _, report = _sharded_complete(mobs_local, mask_local, cfg, last_all, last_off, comm, group,
                                     True)
    return l, report
