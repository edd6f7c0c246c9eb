"""Generate golden vectors from the reference package itself.

Run in the build container (the only place the reference is importable):

    python tests/golden/make_golden.py

It imports ``tenrec`` from /root/reference/pkg/src, runs the reference's own
functions on small seeded inputs and stores inputs + outputs in
``tests/golden/*.npz``.  Nothing at test time reads /root/reference: the
fixtures travel with the repo.  Every case records the reference call it came
from so the oracle and GPU tests can replay it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import tenrec
    from tenrec import onebit, solvers

    out = {}

    # -- penalties: scalar prox on random (mu, v) -------------------------
    pens = {"l1": tenrec.L1(), "firm": tenrec.Firm(gamma=2.5), "mcp": tenrec.MCP(gamma=2.0),
            "scad": tenrec.SCAD(a=3.7), "lq": tenrec.Lq(q=0.5),
            "capped-lq": tenrec.CappedLq(q=0.5, theta=1.0), "log": tenrec.LogPenalty(gamma=1.0)}
    rng = np.random.default_rng(1234)
    mus = rng.uniform(0.01, 5.0, size=64)
    vs = rng.uniform(-10.0, 10.0, size=(64, 33))
    vs[:, 0] = 0.0
    out["prox_mu"] = mus
    out["prox_v"] = vs
    for name, p in pens.items():
        out[f"prox_{name}"] = np.stack([p.prox(float(mu), v) for mu, v in zip(mus, vs)])
        out[f"value_{name}"] = np.stack([p.value(np.abs(v), float(mu)) for mu, v in zip(mus, vs)])
    for q in (0.3, 0.7, 1.0):  # Lq beyond the default exponent
        out[f"prox_lq{q}"] = np.stack([tenrec.Lq(q=q).prox(float(mu), v) for mu, v in zip(mus, vs)])

    # -- structured shrinkage ---------------------------------------------
    a = rng.standard_normal((5, 4, 6, 2))
    out["gnhtt_in"] = a
    for st in ("entry", "tube", "slice"):
        out[f"gnhtt_{st}"] = tenrec.gnhtt(a, tenrec.MCP(2.0), 0.9, st)

    # -- transforms ---------------------------------------------------------
    x = rng.standard_normal((4, 3, 5, 3))
    mats = [np.linalg.qr(rng.standard_normal((n, n)))[0] * np.sqrt(1.0 + i)
            for i, n in enumerate((5, 3))]
    out["tr_in"] = x
    out["tr_mat0"] = mats[0]
    out["tr_mat1"] = mats[1]
    for kind, t in (("fft", tenrec.Transform.fft()), ("dct", tenrec.Transform.dct()),
                    ("explicit", tenrec.Transform.explicit(mats))):
        out[f"tr_{kind}"] = t.apply(x)
        out[f"tr_{kind}_rho"] = np.array(t.rho(x.shape))

    # -- deterministic GNHTSVT ---------------------------------------------
    cases = [((8, 6, 5), "mcp", 0.4), ((10, 8, 4), "l1", 0.6), ((6, 7, 3, 4), "scad", 0.5),
             ((9, 9, 6), "lq", 0.3), ((7, 5, 4), "log", 0.3)]
    for i, (dims, pname, tau) in enumerate(cases):
        a = rng.standard_normal(dims)
        out[f"svt{i}_in"] = a
        out[f"svt{i}_pen"] = np.array(pname)
        out[f"svt{i}_tau"] = np.array(tau)
        out[f"svt{i}_fft"] = tenrec.gnhtsvt(a, tenrec.Transform.fft(), pens[pname], tau)
        out[f"svt{i}_dct"] = tenrec.gnhtsvt(a, tenrec.Transform.dct(), pens[pname], tau)

    # -- randomized GNHTSVT (BKI Tucker compression of modes 0,1) -----------
    # record the reference's own Gaussian draws so a caller can replay them
    rcases = [
        # dims, ranks, blocks, krylov, seed, lowrank, pen, tau
        ((40, 36, 8), (10, 9), None, (3, 3), 0, 6, "mcp", 0.5),
        ((30, 32, 6), (8, 8), (3, 3), (3, 3), 7, 0, "mcp", 0.3),
        ((24, 20, 4, 3), (6, 6), (2, 3), (3, 2), 3, 0, "l1", 0.2),
        ((50, 40, 10), (12, 10), (4, 5), (2, 1), 11, 8, "scad", 0.4),
        ((16, 64, 5), (16, 12), (4, 4), (3, 2), 5, 0, "mcp", 0.2),
    ]
    for i, (dims, ranks, blocks, krylov, seed, lr, pname, tau) in enumerate(rcases):
        if lr:
            facs = [rng.standard_normal((dims[0], lr)), rng.standard_normal((dims[1], lr))]
            core = rng.standard_normal((lr, lr) + dims[2:])
            a = tenrec.mode_product(tenrec.mode_product(core, facs[0], 0), facs[1], 1)
        else:
            a = rng.standard_normal(dims)
        sk = tenrec.SketchConfig(mode="fixed-rank", ranks=ranks, blocks=blocks, krylov=krylov,
                                 seed=seed)
        res = tenrec.gnhtsvt_randomized(a, tenrec.Transform.fft(), pens[pname], tau, sk)
        tf = tenrec.rsthosvd_bki(a, ranks, order=(0, 1), blocks=blocks, krylov=krylov,
                                 seed=seed, strict_rank=False)
        bl = blocks or tuple(max(1, int(np.ceil(r / 4))) for r in ranks)
        g = np.random.default_rng(seed)
        nf = int(np.prod(dims[2:]))
        g0 = g.standard_normal((dims[1] * nf, bl[0]))
        g1 = g.standard_normal((tf.ranks[0] * nf, bl[1]))
        pre = f"rsvt{i}_"
        out[pre + "in"] = a
        out[pre + "ranks"] = np.array(ranks)
        out[pre + "blocks"] = np.array(bl)
        out[pre + "krylov"] = np.array(krylov)
        out[pre + "seed"] = np.array(seed)
        out[pre + "pen"] = np.array(pname)
        out[pre + "tau"] = np.array(tau)
        out[pre + "lowrank"] = np.array(lr)
        out[pre + "out"] = res
        out[pre + "f0"] = tf.factors[0]
        out[pre + "f1"] = tf.factors[1]
        out[pre + "core"] = tf.core
        out[pre + "g0"] = g0
        out[pre + "g1"] = g1

    # -- gradients and the FFT solve ----------------------------------------
    b = rng.standard_normal((8, 7, 5))
    gm = {k: rng.standard_normal(b.shape) for k in (0, 1, 2)}
    gs = tenrec.GradientSet(b.shape, (0, 1, 2))
    out["solve_b"] = b
    for k in (0, 1, 2):
        out[f"solve_g{k}"] = gm[k]
        out[f"grad{k}"] = tenrec.grad(b, k)
        out[f"gradT{k}"] = tenrec.grad_adjoint(b, k)
    out["solve_out"] = tenrec.solve_grad_system(b, gm, gs)
    gs2 = tenrec.GradientSet((6, 5, 4, 3), (0, 3))
    b2 = rng.standard_normal((6, 5, 4, 3))
    gm2 = {0: rng.standard_normal(b2.shape), 3: rng.standard_normal(b2.shape)}
    out["solve2_b"] = b2
    out["solve2_g0"] = gm2[0]
    out["solve2_g3"] = gm2[3]
    out["solve2_out"] = tenrec.solve_grad_system(b2, gm2, gs2)

    # -- ADMM runs (short) ----------------------------------------------------
    truth = tenrec.synth_lowrank_smooth((12, 10, 6), (3, 3, 2), 0.7, 0)
    mobs, mask, _ = tenrec.corrupt(truth, 0.6, 0.1, 1)
    out["admm_truth"] = truth
    out["admm_mobs"] = mobs
    out["admm_mask"] = mask
    for tag, kw in (("det", {}),
                    ("rnd", {"randomized": True,
                             "sketch": tenrec.SketchConfig(mode="fixed-rank", order=(0, 1),
                                                           ranks=(6, 5), blocks=(2, 2),
                                                           krylov=(2, 2), seed=3)}),
                    ("tube", {"structure": "tube", "psi": tenrec.L1()}),
                    ("pure", {"pure_lowrank": True})):
        cfg = tenrec.SolverConfig(max_iters=15, **kw)
        l, e, rep = tenrec.gnrhtc(mobs, mask, cfg)
        out[f"admm_{tag}_l"] = l
        out[f"admm_{tag}_e"] = e
        out[f"admm_{tag}_res"] = np.array(rep.residual_history)
        out[f"admm_{tag}_dfro"] = np.array(rep.diff_fro_history)
        out[f"admm_{tag}_mult"] = np.array(rep.multiplier_history)
    cfg = tenrec.SolverConfig(max_iters=15)
    l, rep = tenrec.gnhtc(mobs, mask, cfg)
    out["admm_nf_l"] = l
    out["admm_nf_res"] = np.array(rep.residual_history)

    # -- one-bit --------------------------------------------------------------
    truth1 = tenrec.synth_lowrank_smooth((10, 9, 5), (3, 3, 2), 0.7, 2)
    obs = tenrec.onebit_observe(truth1, m=900, theta=1.5, sigma=0.1, seed=4, sparse_ratio=0.0)
    out["ob_idx"] = obs.indices
    out["ob_sgn"] = obs.signs
    out["ob_theta"] = np.array(obs.theta)
    out["ob_j1"] = obs.j1
    out["ob_j2"] = obs.j2
    cfg = tenrec.SolverConfig.one_bit(max_iters=12)
    l, rep = tenrec.gnobhtc(obs, cfg)
    out["ob_l"] = l
    out["ob_res"] = np.array(rep.residual_history)
    cfg = tenrec.SolverConfig.one_bit(max_iters=12, lam2=0.05, psi=tenrec.L1())
    l, s, rep = tenrec.gnobrhtc(obs, cfg)
    out["obr_l"] = l
    out["obr_s"] = s
    out["obr_res"] = np.array(rep.residual_history)
    del onebit, solvers

    # -- fixed-accuracy block Lanczos (ad_rsthosvd_blbp) and other orders ------
    # (a separate generator: the cases above stay bit-identical)
    rng2 = np.random.default_rng(2468)
    bcases = [
        # dims, lowrank (0 = none), noise, eps, block, defl_tol, order, seed
        ((14, 12, 6), 3, 1e-3, 0.1, 3, None, None, 5),
        ((16, 18, 5), 4, 0.0, 0.05, 4, None, (1, 0), 9),
        ((12, 10, 4, 3), 0, 0.0, 0.3, 5, None, (0, 1), 2),
        ((20, 8, 6), 2, 1e-2, 0.02, 3, 1e-6, (0, 2, 1), 13),
        ((40, 30, 6), 0, 0.0, 0.2, 4, None, (0, 1), 21),
    ]
    for i, (dims, lr, noise, eps, block, dtol, order, seed) in enumerate(bcases):
        if lr:
            core = rng2.standard_normal((lr,) * len(dims))
            a = core
            for k, n in enumerate(dims):
                a = tenrec.mode_product(a, rng2.standard_normal((n, lr)), k)
            a = a + noise * rng2.standard_normal(dims)
        else:
            a = rng2.standard_normal(dims)
        tf, diag = tenrec.ad_rsthosvd_blbp(a, eps, block=block, defl_tol=dtol, order=order,
                                           seed=seed)
        pre = f"blbp{i}_"
        out[pre + "in"] = a
        out[pre + "eps"] = np.array(eps)
        out[pre + "block"] = np.array(block)
        out[pre + "defl_tol"] = np.array(-1.0 if dtol is None else dtol)
        out[pre + "order"] = np.array(order if order is not None else tuple(range(len(dims))))
        out[pre + "seed"] = np.array(seed)
        out[pre + "core"] = tf.core
        for k, f in enumerate(tf.factors):
            if f is not None:
                out[pre + f"f{k}"] = f
        for name in ("energy_estimates", "ranks", "deflations", "orth_loss", "iterations"):
            d = getattr(diag, name)
            out[pre + name] = np.array([d[k] for k in sorted(d)], dtype=np.float64)
        sk = tenrec.SketchConfig(mode="fixed-accuracy", order=order, eps=eps, block=block,
                                 defl_tol=dtol, seed=seed)
        if len(dims) >= 3:
            out[pre + "svt"] = tenrec.gnhtsvt_randomized(a, tenrec.Transform.fft(), pens["mcp"],
                                                         0.3, sk)
    # fixed-rank compression of every mode / other orders (reference PCG64 draws)
    ocases = [((12, 11, 7), (4, 4, 3), None, None, 3),
              ((10, 12, 6), (5, 4), (1, 0), (2, 2), 8),
              ((9, 10, 8, 3), (4, 3, 3), (2, 0, 1), (3, 2, 1), 4)]
    for i, (dims, ranks, order, blocks, seed) in enumerate(ocases):
        a = rng2.standard_normal(dims)
        tf = tenrec.rsthosvd_bki(a, ranks, order=order, blocks=blocks, krylov=None, seed=seed,
                                 strict_rank=False)
        pre = f"ord{i}_"
        out[pre + "in"] = a
        out[pre + "ranks"] = np.array(ranks)
        out[pre + "order"] = np.array(order if order is not None else tuple(range(len(dims))))
        out[pre + "blocks"] = np.array(blocks if blocks is not None
                                       else tuple(max(1, int(np.ceil(r / 4))) for r in ranks))
        out[pre + "seed"] = np.array(seed)
        out[pre + "core"] = tf.core
        for k, f in enumerate(tf.factors):
            if f is not None:
                out[pre + f"f{k}"] = f
        sk = tenrec.SketchConfig(mode="fixed-rank", order=order or tuple(range(len(dims))),
                                 ranks=ranks, blocks=blocks, seed=seed)
        out[pre + "svt"] = tenrec.gnhtsvt_randomized(a, tenrec.Transform.fft(), pens["mcp"], 0.3,
                                                     sk)

    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
