"""The sharded randomized t-SVT (tr_gnhtsvt_randomized_sharded) against the
single-GPU one.

Two ranks are emulated on the one GPU of the test box by two host threads,
each driving its shard on its own stream; their all-reduce is an in-process
host rendezvous (stream sync, sum in rank order, copy back), so device kernels
never wait on each other.  A world-1 run goes through the production
DeviceAllreduce over a real torch.distributed NCCL group.
"""

import ctypes
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Rendezvous:
    def __init__(self, n):
        self.n = n
        self.barrier = threading.Barrier(n)
        self.slots = [None] * n


class _ThreadAllreduce:
    """tr_allreduce_fn for rank `rank` of an in-process group (test double)."""

    def __init__(self, rv, rank):
        from paper_2506_09594_b200 import _lib

        self.rv, self.rank, self.calls, self.error = rv, rank, 0, None
        self.fn = _lib.ALLREDUCE_FN(self._cb)

    def _cb(self, buf, count, stream, user):
        import torch

        from paper_2506_09594_b200.shard import _CudaArray
        try:
            ptr = ctypes.cast(buf, ctypes.c_void_p).value
            t = torch.as_tensor(_CudaArray(ptr, count), device="cuda")
            torch.cuda.ExternalStream(int(stream or 0)).synchronize()
            self.rv.slots[self.rank] = t
            self.rv.barrier.wait()
            if self.rank == 0:
                acc = self.rv.slots[0].clone()
                for r in range(1, self.rv.n):
                    acc += self.rv.slots[r]
                for r in range(self.rv.n):
                    self.rv.slots[r].copy_(acc)
                torch.cuda.synchronize()
            self.rv.barrier.wait()
            self.calls += 1
            return 0
        except Exception as exc:  # pragma: no cover - surfaced by the caller
            self.error = exc
            self.rv.barrier.abort()
            return 1


def _run_sharded(x, bounds, sketch, tau, dtype):
    import torch

    import paper_2506_09594_b200 as pk
    rv = _Rendezvous(len(bounds))
    outs, errs, reducers = [None] * len(bounds), [], []

    def rank_main(r):
        try:
            off, cnt = bounds[r]
            red = _ThreadAllreduce(rv, r)
            reducers.append(red)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                xl = torch.from_numpy(np.ascontiguousarray(x[..., off:off + cnt])).to(dtype).cuda()
                o = pk.gnhtsvt_randomized_sharded(xl, x.shape[-1], off, pk.Transform.fft(),
                                                  pk.MCP(2.5), tau, sketch, allreduce=red)
                outs[r] = o.double().cpu().numpy()
        except Exception as exc:
            errs.append(exc)
            rv.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(len(bounds))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    # 4 Krylov blocks + Gram per unfolding, 2 unfoldings, + the core
    assert all(red.calls == 2 * (1 + 2 + 1) + 1 for red in reducers)
    return np.concatenate(outs, axis=-1)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_two_shards_match_single_gpu(cuda_lib, dt):
    import torch

    import paper_2506_09594_b200 as pk
    rng = np.random.default_rng(11)
    dims = (64, 48, 12)
    x = rng.standard_normal(dims)
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(8, 8), blocks=(4, 4),
                         krylov=(2, 2), seed=5)
    tau = 0.3
    dtype = torch.float64 if dt == "f64" else torch.float32
    single = pk.gnhtsvt_randomized(torch.from_numpy(x).to(dtype).cuda(), pk.Transform.fft(),
                                   pk.MCP(2.5), tau, sk).double().cpu().numpy()
    for shard_sizes in ([7, 5], [6, 6]):
        bounds, off = [], 0
        for c in shard_sizes:
            bounds.append((off, c))
            off += c
        sharded = _run_sharded(x, bounds, sk, tau, dtype)
        err = np.abs(sharded - single).max() / np.abs(single).max()
        assert err < (1e-10 if dt == "f64" else 1e-4), (shard_sizes, err)


def test_world1_nccl_group_equals_single(cuda_lib):
    import socket

    import torch
    import torch.distributed as dist

    import paper_2506_09594_b200 as pk
    rng = np.random.default_rng(3)
    x = rng.standard_normal((48, 40, 8))
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(6, 6), blocks=(3, 3),
                         krylov=(1, 1), seed=9)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        red = pk.DeviceAllreduce()
        out = pk.gnhtsvt_randomized_sharded(x, x.shape[-1], 0, pk.Transform.fft(), pk.MCP(2.5),
                                            0.2, sk, allreduce=red)
        assert red.calls == 2 * (1 + 1 + 1) + 1
    finally:
        dist.destroy_process_group()
    single = pk.gnhtsvt_randomized(x, pk.Transform.fft(), pk.MCP(2.5), 0.2, sk)
    np.testing.assert_allclose(out, single, rtol=0, atol=1e-12 * np.abs(single).max())


def test_shard_bounds_validated(cuda_lib):
    import paper_2506_09594_b200 as pk
    sk = pk.SketchConfig(mode="fixed-rank", order=(0, 1), ranks=(4, 4), blocks=(2, 2),
                         krylov=(1, 1), seed=1)
    x = np.zeros((16, 16, 4))
    with pytest.raises(ValueError, match="outside"):
        pk.gnhtsvt_randomized_sharded(x, 6, 3, pk.Transform.fft(), pk.MCP(2.5), 0.1, sk)
