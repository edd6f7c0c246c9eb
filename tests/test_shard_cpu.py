"""Host logic of the multi-GPU t-SVT on CPU: world_size-2 gloo processes.

Checks the pieces the sharded CUDA path is built from, on CPU tensors:
  * shard_range tiles the last mode exactly, sizes differing by <= 1;
  * the torch.distributed all-reduce adapter sums in place;
  * the decomposition the sharded t-SVT relies on (tr_gnhtsvt_randomized_sharded):
    with the sketch drawn at GLOBAL column indices (Philox, oracle/philox.py)
    the per-rank Krylov partial sums A_r G_r and A_r A_r^T P, all-reduced, equal
    the unsharded products, and a zero-padded core summed over ranks is the
    whole core.
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, q):
    import torch
    import torch.distributed as dist

    from oracle import philox
    from paper_2506_09594_b200.shard import allreduce_tensor, shard_range
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        n1, n2, n3 = dims
        b = 3
        rng = np.random.default_rng(0)  # same full tensor on every rank
        A = rng.standard_normal((n1, n2 * n3))  # mode-0 unfolding, columns i2 + n2 * i3
        off, cnt = shard_range(n3, world, rank)
        cols = np.arange(n2 * off, n2 * (off + cnt))
        # sketch rows at global column indices, exactly as the CUDA path draws them
        G_local = philox.gaussian_flat(7, 0, (cols[:, None] * b + np.arange(b)).ravel())
        G_local = G_local.reshape(len(cols), b)
        Y = torch.from_numpy(A[:, cols] @ G_local)
        allreduce_tensor(Y)
        P = np.linalg.qr(Y.numpy())[0]
        Z = torch.from_numpy(A[:, cols] @ (A[:, cols].T @ P))
        allreduce_tensor(Z)
        core = np.zeros((2, 2, n3))
        core[:, :, off:off + cnt] = rank + 1.0
        core_t = torch.from_numpy(core)
        allreduce_tensor(core_t)
        t = torch.full((4,), float(rank + 1), dtype=torch.float64)
        allreduce_tensor(t)
        q.put((rank, off, cnt, Y.numpy(), Z.numpy(), core_t.numpy(), t.numpy(), None))
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover
        q.put((rank, None, None, None, None, None, None, repr(exc)))


def test_shard_range_tiles_exactly():
    from paper_2506_09594_b200.shard import shard_range
    for n in (1, 5, 12, 128, 131):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, world, r) for r in range(world)]
            assert parts[0][0] == 0
            for (o1, c1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + c1 == o2
            assert sum(c for _, c in parts) == n
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_gloo_world2_sharded_decomposition():
    import multiprocessing as mp

    from oracle import philox
    dims = (20, 6, 7)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env_pp = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = root + (os.pathsep + env_pp if env_pp else "")
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    try:
        for p in procs:
            p.start()
        res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    finally:
        for p in procs:
            p.join(timeout=60)
        os.environ["PYTHONPATH"] = env_pp
    for r in res:
        assert r[-1] is None, r[-1]
    n1, n2, n3 = dims
    b = 3
    A = np.random.default_rng(0).standard_normal((n1, n2 * n3))
    G = philox.gaussian_flat(7, 0, np.arange(n2 * n3 * b)).reshape(n2 * n3, b)
    Y_full = A @ G
    P = np.linalg.qr(Y_full)[0]
    Z_full = A @ (A.T @ P)
    for rank, off, cnt, Y, Z, core, t, _ in res:
        np.testing.assert_allclose(Y, Y_full, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(Z, Z_full, rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(t, np.full(4, 3.0))
        expect = np.zeros((2, 2, n3))
        for r2, o2, c2, *_ in res:
            expect[:, :, o2:o2 + c2] = r2 + 1.0
        np.testing.assert_allclose(core, expect)
    assert [(r[1], r[2]) for r in res] == [(0, 4), (4, 3)]
