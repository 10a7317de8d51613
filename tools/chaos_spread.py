"""How far the full-size trajectories' agreement spans spread under
last-bit perturbations (GPU).  For each config, the device runs the
fixture's pair unchanged and K times with the least significant bit of the
moving image flipped at a random half of its voxels (a relative input
change of <= 6e-8, the size of the fp32 rounding every storage point
applies), and reports the first iteration at which each run's loss leaves
the pure fp64 oracle's by more than 1e-5 (the north-star bar), next to the
fp32-storage oracle's own span: the spread of the span over equally good
fp32-storage trajectories.

    python tools/chaos_spread.py [K] [config ...] > profiles/r02/chaos_spread.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from golden.make_fullsize import CASES, pair  # noqa: E402
from fullsize_parity import gpu_run  # noqa: E402


def first_div(a, b, tol=1e-5):
    n = min(len(a), len(b))
    rel = np.abs(a[:n, 2] - b[:n, 2]) / np.abs(b[:n, 2])
    return next((int(k) for k in range(n) if rel[k] > tol), n)


def main():
    import paper_2603_19371_b200 as P
    args = sys.argv[1:]
    K = int(args.pop(0)) if args and args[0].isdigit() else 8
    names = args or ["config2", "config3_lm", "config4"]
    ctx = P.Context(0)
    out = {}
    for name in names:
        fx = np.load(os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz"))
        o64, o32 = fx["fp64_trace"], fx["fp32_trace"]
        idx, w64 = fx["sample_idx"], fx["fp64_warp_s"]

        def wrel(warp):
            w = warp.reshape(-1, 3)[idx]
            return float(np.linalg.norm(w - w64) / np.linalg.norm(w64))

        F, M = pair(name)
        tr, warp = gpu_run(name, F, M, ctx)
        rng = np.random.default_rng(7)
        spans, wd = [], []
        for k in range(K):
            Mp = M.copy()
            flat = Mp.reshape(-1).view(np.uint32)
            flat ^= rng.integers(0, 2, size=flat.size, dtype=np.uint32)
            trp, wp = gpu_run(name, F, Mp, ctx)
            spans.append(first_div(trp, o64))
            wd.append(wrel(wp))
        out[name] = {"iterations": int(len(o64)),
                     "storage_oracle_vs_fp64": first_div(o32, o64),
                     "device_vs_fp64": first_div(tr, o64),
                     "perturbed_device_vs_fp64": spans,
                     "perturbed_min_median_max": [int(min(spans)), float(np.median(spans)), int(max(spans))],
                     "warp_rel_l2_vs_fp64": {"storage_oracle": float(np.linalg.norm(fx["fp32_warp_s"] - w64) /
                                                                     np.linalg.norm(w64)),
                                             "device": wrel(warp), "perturbed": wd,
                                             "perturbed_min_median_max": [min(wd), float(np.median(wd)), max(wd)]}}
        print(name, json.dumps(out[name]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
