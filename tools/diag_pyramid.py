"""Diagnostic: register() pyramid, GPU vs oracle, per-iteration divergence."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2603_19371_b200 as P
ctx = P.Context(0)
F, M, _ = O.synth_pair((40, 48, 56), 1, num_blobs=10, warp_max=4.0)
rej = int(sys.argv[1]) if len(sys.argv) > 1 else 1
kw = dict(nlevels=3, factors=[4, 2, 1], iters=[30, 20, 10])
res = P.register(F, M, P.reg_config(**kw, **{"lm.rejection": rej}), ctx=ctx)
rc, w_o, tr_o, jac_o = O.register(F, M, O.default_config(**kw, **{"lm.rejection": rej}))
for a, b in zip(res.loss_trace, tr_o):
    print("L%d it%2d r %.6f rel %.2e eps rel %.2e acc %d/%d ret %d/%d lam %s" % (
        a.level, a.iter, b.r, abs(a.r - b.r) / b.r, abs(a.eps - b.eps) / b.eps, a.accepted, b.accepted,
        a.retries, b.retries, a.lam == b.lam))
print("warp rel", np.linalg.norm(res.final_warp - w_o) / np.linalg.norm(w_o))
for f in (4, 2):
    d = P.downsample(F.astype(np.float64), f, ctx=ctx)
    do = O.downsample(F.astype(np.float64), f).astype(np.float32)
    print("downsample f=%d max abs diff vs fp32-rounded oracle: %.3e (ulps: %d)" % (
        f, np.abs(d - do).max(), int((d.astype(np.float32).view(np.int32) - do.view(np.int32)).__abs__().max())))
