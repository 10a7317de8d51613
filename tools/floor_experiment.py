"""The fp32-storage floor of the LM trajectory (CPU, oracle only).

Runs the fp64 oracle twice on the same pair: once in pure fp64 and once with
the warp rounded to fp32 after every iteration (what any fp32-storage
implementation must at least do).  The divergence between the two is the
floor no fp32 device path can beat; it sets the parity bars in DESIGN.md.

    PYTHONPATH=. python tools/floor_experiment.py [--small]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402


def run(F, M, iters, fp32_state):
    cfg = O.default_config(nlevels=1, factors=[1], iters=[1])
    u = np.zeros(F.shape + (3,))
    st = O.LmState(0.006, 0, 0.0, 0.0)
    rs = []
    for _ in range(iters):
        rc, u, st, tr = O.lm_run_level(F, M, u, cfg, 1, state=st)
        rs.append(tr[0].r)
        if fp32_state:
            u = u.astype(np.float32).astype(np.float64)
    return np.array(rs), u


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true", help="10x12x14 coarse pyramid level")
    ap.add_argument("--seeds", type=int, nargs="*", default=[0, 1, 2])
    a = ap.parse_args()
    for seed in a.seeds:
        if a.small:
            F, M, _ = O.synth_pair((40, 48, 56), seed, num_blobs=10, warp_max=4.0)
            F = O.downsample(F.astype(np.float64), 4).astype(np.float32).astype(np.float64)
            M = O.downsample(M.astype(np.float64), 4).astype(np.float32).astype(np.float64)
            iters = 30
        else:
            F, M, _ = O.synth_pair((64, 64, 64), seed, num_blobs=12, warp_max=3.0)
            iters = 100
        r64, u64 = run(F, M, iters, False)
        r32, u32 = run(F, M, iters, True)
        d = np.abs(r32 - r64) / r64
        first = next((i for i, x in enumerate(d) if x > 1e-6), None)
        print(f"seed {seed} shape {F.shape}: max loss rel {d.max():.2e} (first > 1e-6 at iter {first}), "
              f"final warp rel-L2 {np.linalg.norm(u32 - u64) / np.linalg.norm(u64):.2e}", flush=True)


if __name__ == "__main__":
    main()
