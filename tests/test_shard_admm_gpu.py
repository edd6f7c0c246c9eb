"""The multi-GPU ADMM (tr_admm_create_sharded; BASELINE configs[4]'s path) on
the one test GPU.

Every rank of a sharded solve must see the same sweep as the unsharded solver:
the distributed FFT solve (all-to-all transpose of the last axis), the ghost
faces of the circular stencils and the last-mode-sharded t-SVTs change only
fp64 summation order.  Two ranks run as two processes sharing the GPU, joined
by gloo (collectives staged through host memory -- NCCL cannot put two ranks on
one device); world 1 runs the same code path in-process with local exchanges.
Both are compared with the single-GPU solver on the whole tensor.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _problem(dims, seed=3):
    rng = np.random.default_rng(seed)
    r = 3
    x = rng.standard_normal((r,) * len(dims))
    for k, n in enumerate(dims):
        x = np.moveaxis(np.tensordot(rng.standard_normal((n, r)), x, axes=([1], [k])), 0, k)
    x /= np.abs(x).max()
    mask = rng.random(dims) < 0.6
    out = rng.random(dims) < 0.05
    mobs = np.where(out, rng.uniform(-1, 1, dims), x)
    return np.where(mask, mobs, 0.0), mask


def _cfg(pk, iters, ranks=(5, 5), blocks=(2, 2), krylov=(2, 2), seed=4):
    sk = pk.SketchConfig(mode="fixed-rank", ranks=ranks, blocks=blocks, krylov=krylov, seed=seed)
    return pk.SolverConfig(randomized=True, sketch=sk, max_iters=iters, tol=1e-30)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dims", [(32, 24, 8), (16, 12, 4, 8)])
def test_world1_sharded_matches_unsharded(cuda_lib, dims):
    import torch.distributed as dist

    import paper_2506_09594_b200 as pk

    mobs, mask = _problem(dims)
    cfg = _cfg(pk, 5)
    l0, e0, r0 = pk.gnrhtc(mobs, mask, cfg)
    own = not dist.is_initialized()
    if own:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1)
    try:
        l1, e1, r1 = pk.gnrhtc_sharded(mobs, mask, cfg, dims[-1], 0)
    finally:
        if own:
            dist.destroy_process_group()
    assert _rel(l1, l0) <= 1e-12 and _rel(e1, e0) <= 1e-12
    np.testing.assert_allclose(np.array(r1.residual_history), np.array(r0.residual_history),
                               rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("dims,dtype,noise_free", [
    ((32, 24, 8), "f64", False),
    ((16, 12, 4, 8), "f64", False),
    ((16, 12, 4, 8), "f64", True),
    ((32, 24, 8), "f32", False),
])
def test_two_ranks_match_single_gpu(cuda_lib, tmp_path, dims, dtype, noise_free):
    import paper_2506_09594_b200 as pk

    mobs, mask = _problem(dims)
    iters, ranks, blocks, krylov, seed = 5, (5, 5), (2, 2), (2, 2), 4
    prob = tmp_path / "prob.npz"
    np.savez(prob, mobs=mobs, mask=mask, dtype=dtype, ranks=ranks, blocks=blocks, krylov=krylov,
             seed=seed, iters=iters, noise_free=noise_free)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "shard_admm_worker.py"),
                               str(prob), str(tmp_path / f"r{r}.npz"), str(r), str(world),
                               str(port)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out.decode()[-3000:]
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    l = np.concatenate([p["l"] for p in parts], axis=-1)
    e = np.concatenate([p["e"] for p in parts], axis=-1)
    x = mobs.astype(np.float32) if dtype == "f32" else mobs
    cfg = _cfg(pk, iters, ranks, blocks, krylov, seed)
    if noise_free:
        l0, r0 = pk.gnhtc(x, mask, cfg)
    else:
        l0, e0, r0 = pk.gnrhtc(x, mask, cfg)
        assert _rel(e, e0) <= (1e-9 if dtype == "f64" else 1e-4)
    tol = 1e-9 if dtype == "f64" else 1e-4
    assert _rel(l, l0) <= tol, _rel(l, l0)
    for p in parts:  # every rank reports the global residuals
        np.testing.assert_allclose(p["res"], np.array(r0.residual_history),
                                   rtol=1e-7 if dtype == "f64" else 1e-3, atol=1e-12)
        np.testing.assert_allclose(p["mult"], np.array(r0.multiplier_history),
                                   rtol=1e-7 if dtype == "f64" else 1e-3)
