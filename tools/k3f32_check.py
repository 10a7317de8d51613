"""Config 1 (64^3 x 100, seeds 0-2) with the library under WLM_LIB_PATH against
the pure fp64 oracle and the oracle's "K3hilo" precision mode (fp32 K3 with
hi/lo weights, tools/precision_modes.py).  GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2603_19371_b200 as P

ctx = P.Context(0)
for seed in (0, 1, 2):
    F, M, _ = O.synth_pair((64, 64, 64), seed, num_blobs=12, warp_max=3.0)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[100])
    e = P.Engine(F.shape, 1, cfg, ctx=ctx)
    e.load(F[None], M[None]); e.set_warp(None); e.begin_level(0); e.iterate(100)
    r = np.array([t["r"] for t in e.trace(0)]); w = np.moveaxis(e.get_warp()[0].astype(np.float64), 0, -1)
    e.close()
    co = O.default_config(nlevels=1, factors=[1], iters=[100])
    out = []
    for name, mode, flags in (("fp64", 0, 3), ("storage", 1, 3), ("K3hilo", 2, 1 | 8 | 16)):
        L = O.lib(); L.orc_set_fp32_storage(mode); L.orc_set_dev_flags(flags)
        try:
            rc, u, st, tr = O.lm_run_level(F, M, np.zeros(F.shape + (3,)), co, 100)
        finally:
            L.orc_set_fp32_storage(0); L.orc_set_dev_flags(3)
        ro = np.array([t.r for t in tr])
        d = np.abs(r - ro) / ro
        out.append(f"{name}: max loss {d.max():.2e} warp {np.linalg.norm(w - u) / np.linalg.norm(u):.2e}")
    print(f"seed {seed}: " + "; ".join(out), flush=True)
