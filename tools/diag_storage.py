"""Diagnostic: GPU vs the fp64 oracle and vs the fp32-storage oracle, for the
configurations the parity tests use.  Prints max per-iteration loss relative
deviation, accept/retry agreement, lambda agreement and final warp rel-L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2603_19371_b200 as P  # noqa: E402

ctx = P.Context(0)


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


def stats(name, tr, tr_o, w, w_o):
    r = [t["r"] if isinstance(t, dict) else t.r for t in tr]
    acc = [(t["accepted"], t["retries"]) if isinstance(t, dict) else (t.accepted, t.retries) for t in tr]
    lam = [t["lam"] if isinstance(t, dict) else t.lam for t in tr]
    d = [abs(a - b.r) / b.r for a, b in zip(r, tr_o)]
    same_acc = acc == [(b.accepted, b.retries) for b in tr_o]
    same_lam = lam == [b.lam for b in tr_o]
    first_bad = next((i for i, x in enumerate(d) if x > 1e-5), None)
    print(f"{name:34s} n={len(d):3d} maxrel={max(d):.2e} first>1e-5={first_bad} acc_eq={same_acc} "
          f"lam_eq={same_lam} warp={rel(w, w_o):.2e}", flush=True)


def engine_run(F, M, cfg, iters):
    eng = P.Engine(F.shape, 1, cfg, ctx=ctx)
    eng.load(F[None], M[None]); eng.set_warp(None); eng.begin_level(0); eng.iterate(iters)
    w = np.moveaxis(eng.get_warp()[0].astype(np.float64), 0, -1)
    tr = eng.trace(0)
    eng.close()
    return tr, w


cases = [
    ("config1 64^3 x100", (64, 64, 64), 0, 12, 3.0, {}, 100),
    ("rejection 32x36x40 x40 tau0.2", (32, 36, 40), 3, 10, 3.0, {"lm.rejection": 1, "lm.tau": 0.2}, 40),
    ("adam 24^3 x20", (24, 24, 24), 8, 6, 2.0, {"optimizer": P.OPT_ADAM}, 20),
    ("gd 24^3 x20", (24, 24, 24), 8, 6, 2.0, {"optimizer": P.OPT_GD, "gd_lr": 2.0}, 20),
]
for name, shape, seed, blobs, wm, kw, iters in cases:
    F, M, _ = O.synth_pair(shape, seed, num_blobs=blobs, warp_max=wm)
    tr, w = engine_run(F, M, P.reg_config(nlevels=1, factors=[1], iters=[iters], **kw), iters)
    cfg_o = O.default_config(nlevels=1, factors=[1], iters=[iters], **kw)
    for mode in ("fp64", "fp32-storage"):
        if mode == "fp32-storage":
            O.lib().orc_set_fp32_storage(1)
        rc, u_o, _, tr_o = O.lm_run_level(F, M, np.zeros(shape + (3,)), cfg_o, iters)
        O.lib().orc_set_fp32_storage(0)
        stats(f"{name} vs {mode}", tr, tr_o, w, u_o)

F, M, _ = O.synth_pair((40, 48, 56), 1, num_blobs=10, warp_max=4.0)
kw = dict(nlevels=3, factors=[4, 2, 1], iters=[30, 20, 10])
res = P.register(F, M, P.reg_config(**kw, **{"lm.rejection": 1}), ctx=ctx)
for mode in ("fp64", "fp32-storage"):
    if mode == "fp32-storage":
        O.lib().orc_set_fp32_storage(1)
    rc, w_o, tr_o, jac_o = O.register(F, M, O.default_config(**kw, **{"lm.rejection": 1}))
    O.lib().orc_set_fp32_storage(0)
    stats(f"pyramid 40x48x56 rej vs {mode}", res.loss_trace, tr_o, res.final_warp, w_o)
