"""Multi-GPU randomized t-SVT: one rank per GPU, the tensor sharded along its
last mode (row (e)).

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

__all__ = ["shard_range", "allreduce_tensor", "DeviceAllreduce", "gnhtsvt_randomized_sharded"]


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
    """Zero-copy __cuda_array_interface__ view of fp64 device memory."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
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
