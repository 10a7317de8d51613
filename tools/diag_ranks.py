"""Two-rank slab transport step by step (debug aid; GPU)."""
import multiprocessing as mp, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_slab_ranks import SHAPE, SHIM, _pair, _unique_id

def rank(r, uid, q):
    import paper_2603_19371_b200 as P
    from paper_2603_19371_b200 import slabs
    F, M = _pair()
    ctx = P.Context(0)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[3])
    g = slabs.RankSlab(SHAPE, r, 2, uid, cfg=cfg, ctx=ctx, nccl_lib=SHIM)
    g.load(F, M); g.set_warp(None)
    out = []
    try:
        g.begin_level(0); out.append(("begin", g.state()))
        for k in range(3):
            g.iterate(1); out.append((k, g.state()))
    except Exception as e:
        out.append(("err", repr(e)))
        try: out.append(("state", g.state()))
        except Exception as e2: out.append(("state-err", repr(e2)))
    q.put((r, out))

if __name__ == "__main__":
    import paper_2603_19371_b200 as P
    F, M = _pair()
    ctx = P.Context(0)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[3])
    e = P.Engine(SHAPE, 1, cfg, ctx=ctx); e.load(F[None], M[None]); e.set_warp(None); e.begin_level(0)
    print("single begin", e.state(0)); e.iterate(3); print("single", e.state(0))
    uid = _unique_id()
    c = mp.get_context("spawn"); q = c.Queue()
    ps = [c.Process(target=rank, args=(r, uid, q)) for r in range(2)]
    [p.start() for p in ps]
    for _ in range(2):
        r, out = q.get(timeout=120)
        for o in out: print("rank", r, o)
    [p.join() for p in ps]
