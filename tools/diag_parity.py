"""Diagnostic (not a test): per-iteration GPU vs oracle divergence at 64^3."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2603_19371_b200 as P

def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())

ctx = P.Context(0)
F, M, _ = O.synth_pair((64, 64, 64), 0, num_blobs=12, warp_max=3.0)
F64, M64 = F.astype(np.float64), M.astype(np.float64)
u = np.zeros((64, 64, 64, 3))
rep = P.residual_lncc(F64, M64, u, ctx=ctx)
r, g, ln, I = O.residual_lncc(F64, M64, u, internals=True)
print("iter0 residual: r rel %.3e  g relL2 %.3e  g maxrel %.3e" % (abs(rep.r - r) / r, rel(rep.g, g),
      np.abs(rep.g - g).max() / np.abs(g).max()))
for shift in ("mean",):
    pass
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[N])
eng = P.Engine((64, 64, 64), 1, cfg_p, ctx=ctx)
eng.load(F[None], M[None]); eng.set_warp(None); eng.begin_level(0); eng.iterate(N)
tr = eng.trace(0)
wg = np.moveaxis(eng.get_warp()[0].astype(np.float64), 0, -1)
cfg_o = O.default_config(nlevels=1, factors=[1], iters=[N])
rc, uo, st, tro = O.lm_run_level(F, M, np.zeros((64, 64, 64, 3)), cfg_o, N)
for a, b in zip(tr, tro):
    print("it %3d  r %.9f  rel %.2e  eps rel %.2e  lam eq %s" % (a["iter"], b.r, abs(a["r"] - b.r) / b.r,
          abs(a["eps"] - b.eps) / b.eps, a["lam"] == b.lam))
print("warp relL2 %.3e" % rel(wg, uo))

# ---- per-voxel coefficient comparison at u = 0 ----
eng = P.Engine((64, 64, 64), 1, P.reg_config(nlevels=1, factors=[1], iters=[1]), ctx=ctx)
eng.load(F[None], M[None]); eng.set_warp(None); eng.begin_level(0)
abe = [np.asarray(a, np.float64) for a in eng.read_buffer("abe")]
sf, sm = float(np.float32(F64.mean())), float(np.float32(M64.mean()))
for name, gpu, ref in (("A", abe[0], I.A), ("B", abe[1], I.B), ("E", abe[2], I.E - I.A * sf - I.B * sm)):
    err = np.abs(gpu - ref)
    scale = np.abs(ref).max()
    j = np.unravel_index(err.argmax(), err.shape)
    print("%s: max abs err/scale %.2e at %s, relL2 %.2e, mean signed rel %.2e" % (
        name, err.max() / scale, j, rel(gpu, ref), np.mean((gpu - ref)[ref != 0] / ref[ref != 0])))
eng.close()
