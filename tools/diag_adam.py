import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as O, paper_2603_19371_b200 as P
from golden.make_fullsize import pair
F, M = pair("config3_adam")
Fl = O.downsample(F.astype(np.float64), 8).astype(np.float32)
Ml = O.downsample(M.astype(np.float64), 8).astype(np.float32)
ctx = P.Context(0)
for opt in (1, 0, 2):
    it = 100
    kw = dict(nlevels=1, factors=[1], iters=[it], optimizer=opt)
    if opt == 2: kw["gd_lr"] = 2.0
    eng = P.Engine(Fl.shape, pairs=1, cfg=P.reg_config(**kw), ctx=ctx)
    eng.load(Fl[None], Ml[None]); eng.set_warp(None); eng.begin_level(0); eng.iterate(it)
    tr = eng.trace(0); eng.close()
    res = {}
    for st in ("fp32", "fp64"):
        cfg = O.default_config(**kw)
        if st == "fp32":
            with O.fp32_storage():
                rc, u, s_, tro = O.lm_run_level(Fl, Ml, np.zeros(Fl.shape + (3,)), cfg, it)
        else:
            rc, u, s_, tro = O.lm_run_level(Fl, Ml, np.zeros(Fl.shape + (3,)), cfg, it)
        d = np.array([abs(a["r"] - b.r) / b.r for a, b in zip(tr, tro)])
        res[st] = (d[:5].max(), next((k for k in range(it) if d[k] > 1e-9), None), next((k for k in range(it) if d[k] > 1e-6), None))
    print("opt", opt, Fl.shape, res, flush=True)
