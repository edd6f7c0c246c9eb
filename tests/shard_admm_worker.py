"""One rank of the sharded-ADMM GPU test (tests/test_shard_admm_gpu.py).

python tests/shard_admm_worker.py PROBLEM.npz OUT.npz RANK WORLD PORT

Joins a gloo group on 127.0.0.1 (several ranks may share the one test GPU: the
collectives are staged through host memory), solves its slab of the last mode
with gnrhtc_sharded / gnhtc_sharded and saves its L / E slabs and the (global)
residual history.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    prob, out, rank, world, port = sys.argv[1], sys.argv[2], *map(int, sys.argv[3:6])
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    import paper_2506_09594_b200 as pk

    z = np.load(prob)
    mobs, mask = z["mobs"], z["mask"]
    if str(z["dtype"]) == "f32":
        mobs = mobs.astype(np.float32)
    n = mobs.shape[-1]
    nl = n // world
    sl = (Ellipsis, slice(rank * nl, (rank + 1) * nl))
    sk = pk.SketchConfig(mode="fixed-rank", ranks=tuple(z["ranks"]), blocks=tuple(z["blocks"]),
                         krylov=tuple(z["krylov"]), seed=int(z["seed"]))
    cfg = pk.SolverConfig(randomized=True, sketch=sk, max_iters=int(z["iters"]), tol=1e-30)
    ml, mk = np.asfortranarray(mobs[sl]), np.asfortranarray(mask[sl])
    if bool(z["noise_free"]):
        l, rep = pk.gnhtc_sharded(ml, mk, cfg, n, rank * nl)
        e = np.zeros_like(l)
    else:
        l, e, rep = pk.gnrhtc_sharded(ml, mk, cfg, n, rank * nl)
    np.savez(out, l=l, e=e, res=np.array(rep.residual_history),
             dfro=np.array(rep.diff_fro_history), mult=np.array(rep.multiplier_history))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
