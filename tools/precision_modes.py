"""Which fp32 arithmetic can the device afford?  (CPU, oracle only.)

Runs the oracle's lm_run_level in its precision modes against pure fp64:
  storage   -- fp32 rounding at the device's storage points (mode 1)
  dev32     -- + the K3 step and both Gaussian smoothings in fp32 (mode 2)
  dev32+c   -- + the compositive resample in fp32 (experiment)
and prints the max per-iteration loss deviation and the final warp rel-L2.

    python tools/precision_modes.py [--small] [--seeds 0 1 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402


def run(F, M, iters, mode, flags=3, **kw):
    L = O.lib("port")
    L.orc_set_fp32_storage(mode)
    L.orc_set_dev_flags(flags)
    try:
        cfg = O.default_config(nlevels=1, factors=[1], iters=[iters], **kw)
        rc, u, st, tr = O.lm_run_level(F, M, np.zeros(F.shape + (3,)), cfg, iters)
    finally:
        L.orc_set_fp32_storage(0)
        L.orc_set_dev_flags(3)
    return np.array([t.r for t in tr]), u, [(t.accepted, t.retries) for t in tr]


MODES = [("storage", 1, 0), ("K3f32", 2, 1), ("K4sf32", 2, 2), ("comp32", 2, 4), ("K3+K4s", 2, 3), ("all32", 2, 7), ("K3n64", 2, 1 | 16), ("K3hilo", 2, 1 | 8 | 16), ("K4hilo", 2, 2 | 8), ("all_hilo", 2, 7 | 8 | 16)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true", help="10x12x14 coarse pyramid level")
    ap.add_argument("--seeds", type=int, nargs="*", default=[0, 1, 2])
    ap.add_argument("--rejection", action="store_true")
    ap.add_argument("--modes", nargs="*", default=None)
    a = ap.parse_args()
    kw = {"lm.rejection": 1, "lm.tau": 0.2} if a.rejection else {}
    global MODES
    if a.modes:
        MODES = [m for m in MODES if m[0] in a.modes]
    for seed in a.seeds:
        if a.small:
            F, M, _ = O.synth_pair((40, 48, 56), seed, num_blobs=10, warp_max=4.0)
            F = O.downsample(F.astype(np.float64), 4).astype(np.float32).astype(np.float64)
            M = O.downsample(M.astype(np.float64), 4).astype(np.float32).astype(np.float64)
            iters = 30
        else:
            F, M, _ = O.synth_pair((64, 64, 64), seed, num_blobs=12, warp_max=3.0)
            iters = 100
        r64, u64, d64 = run(F, M, iters, 0, **kw)
        for name, mode, fl in MODES:
            r, u, dec = run(F, M, iters, mode, fl, **kw)
            d = np.abs(r - r64) / r64
            first = next((i for i, x in enumerate(d) if x > 1e-6), None)
            print(f"seed {seed} {F.shape} {name:8s}: max loss rel {d.max():.2e} (first >1e-6 at {first}), "
                  f"warp rel-L2 {np.linalg.norm(u - u64) / np.linalg.norm(u64):.2e}, "
                  f"decisions {'same' if dec == d64 else 'DIFFER'}", flush=True)


if __name__ == "__main__":
    main()
