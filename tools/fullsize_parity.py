"""Full-size parity of BASELINE configs 2, 3 and 4 against the committed
oracle runs (tests/golden/fullsize_*.npz, made by tests/golden/make_fullsize.py).

Prints, per config, against the fp32-storage and the pure fp64 oracle: the
number of iterations, the first iteration whose loss differs by more than
1e-6 / 1e-5 (relative), the first accept/retry/lambda mismatch, the largest
loss deviation, and the final-warp rel-L2 over the fixture's voxel sample;
plus the fp32-storage oracle's own distance from fp64 (the storage floor).

    python tools/fullsize_parity.py [config2 config3_lm config3_adam config4]   (GPU)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden.make_fullsize import CASES, inputs_sha, pair  # noqa: E402


def gpu_run(name, F, M, ctx):
    import paper_2603_19371_b200 as P
    _, _, _, kw = CASES[name]
    cfg = P.reg_config(**kw)
    if kw["nlevels"] == 1:
        # the bench's own path: the batch engine (config 4), one pair
        eng = P.Engine(F.shape, pairs=1, cfg=cfg, ctx=ctx)
        eng.load(F[None], M[None])
        eng.set_warp(None)
        eng.begin_level(0)
        eng.iterate(kw["iters"][0])
        warp = np.moveaxis(eng.get_warp()[0].astype(np.float64), 0, -1)
        tr = np.array([(t["level"], t["iter"], t["r"], t["lam"], t["accepted"], t["retries"])
                       for t in eng.trace(0)])
        eng.close()
        return tr, warp
    res = P.register(F, M, cfg, ctx=ctx)
    tr = np.array([(t.level, t.iter, t.r, t.lam, t.accepted, t.retries) for t in res.loss_trace])
    return tr, res.final_warp


def compare(tr, warp, fx, var, idx):
    o = fx[f"{var}_trace"]
    n = min(len(tr), len(o))
    rel = np.abs(tr[:n, 2] - o[:n, 2]) / np.abs(o[:n, 2])
    dec = [(k) for k in range(n) if tr[k, 4] != o[k, 4] or tr[k, 5] != o[k, 5] or tr[k, 3] != o[k, 3]
           or tr[k, 0] != o[k, 0] or tr[k, 1] != o[k, 1]]
    w = warp.reshape(-1, 3)[idx]
    ws = fx[f"{var}_warp_s"]
    return {"iters_gpu": int(len(tr)), "iters_oracle": int(len(o)),
            "first_loss_gt_1e-6": next((int(k) for k in range(n) if rel[k] > 1e-6), None),
            "first_loss_gt_1e-5": next((int(k) for k in range(n) if rel[k] > 1e-5), None),
            "first_decision_or_lambda_mismatch": dec[0] if dec else None,
            "max_loss_rel": float(rel.max()),
            "warp_rel_l2_sample": float(np.linalg.norm(w - ws) / np.linalg.norm(ws))}


def main():
    import paper_2603_19371_b200 as P
    ctx = P.Context(0)
    out = {}
    for name in sys.argv[1:] or list(CASES):
        fx = np.load(os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz"))
        F, M = pair(name)
        assert inputs_sha(F, M) == str(fx["inputs_sha"]), "inputs differ from the fixture's"
        tr, warp = gpu_run(name, F, M, ctx)
        idx = fx["sample_idx"]
        r = {v: compare(tr, warp, fx, v, idx) for v in ("fp32", "fp64")}
        a, b = fx["fp32_warp_s"], fx["fp64_warp_s"]
        r["storage_floor_warp_rel_l2_sample"] = float(np.linalg.norm(a - b) / np.linalg.norm(b))
        o32, o64 = fx["fp32_trace"], fx["fp64_trace"]
        n = min(len(o32), len(o64))
        rr = np.abs(o32[:n, 2] - o64[:n, 2]) / np.abs(o64[:n, 2])
        dd = [k for k in range(n) if o32[k, 4] != o64[k, 4] or o32[k, 5] != o64[k, 5] or o32[k, 3] != o64[k, 3]]
        r["oracles_first_loss_gt_1e-5"] = next((int(k) for k in range(n) if rr[k] > 1e-5), None)
        r["oracles_first_decision_mismatch"] = dd[0] if dd else None
        out[name] = r
        print(name, json.dumps(r), flush=True)
    return out


if __name__ == "__main__":
    main()
