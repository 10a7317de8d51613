"""Full-size (192^3) parity diagnostic: device vs the fp64 and fp32-storage
oracles after 1 and 4 LM iterations, and the storage floor between them.
Test infrastructure (reads oracle/); run on a GPU box: python tools/diag192.py"""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle as O
import paper_2603_19371_b200 as P
from conftest import rel
from test_gpu_parity import run_engine, oracle_level, aos
F, M, _ = O.synth_pair((192,)*3, 1000, num_blobs=12, warp_max=6.0)
ctx = P.Context(0)
for it in (1, 4):
    cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[it]); cfg_o = O.default_config(nlevels=1, factors=[1], iters=[it])
    warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, it)
    w = aos(warp[0])
    res = {}
    for s in ("fp64", "fp32"):
        rc, u_o, _, tr_o = oracle_level(F, M, cfg_o, it, s)
        res[s] = u_o
        d = np.abs(w - u_o).max(axis=-1)
        print(it, s, "rel", rel(w, u_o), "maxabs", d.max(), "n>1e-3", int((d > 1e-3).sum()), "loss", [ (a.r if not isinstance(a, dict) else a['r']) for a in tr][-1], tr_o[-1].r, flush=True)
    print(it, "floor fp32-oracle vs fp64-oracle rel", rel(res["fp32"], res["fp64"]), flush=True)
