"""Golden oracle runs of BASELINE configs 2, 3 and 4 at their full sizes.

TEST INFRASTRUCTURE.  Runs the fp64 oracle (oracle/liboracle.so, the
restatement pinned to the reference's own field.cpp by tests/test_oracle.py)
on the configs' own synthetic pairs, twice per run: pure fp64, and with the
device's fp32 storage points emulated (orc_set_fp32_storage).  Writes
tests/golden/fullsize_<name>.npz with

  inputs_sha   sha256 of the F and M bytes (the test regenerates the pair
               with the same oracle synth_pair and checks the hash)
  <var>_trace  per accepted iteration: level, iter, r, lambda, accepted,
               retries  (var = fp64 | fp32)
  <var>_warp_s the final warp at a fixed sample of voxels (rounded to fp32,
               the device's storage precision; AoS x, y, z)
  <var>_warp_norm  the whole final warp's L2 norm
  sample_idx   the sampled flat voxel indices (seeded, sorted)

The full warps (80-120 MB each) are not committed; the sample gives the
warp rel-L2 over 2^15 voxels, an unbiased estimate of the whole-volume one.

    python tests/golden/make_fullsize.py [config2 config3_lm config3_adam config4]

CPU only, ~30 min on 8 cores for all four.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

NSAMPLE = 1 << 15

# (name, shape (nz, ny, nx), seed, warp_max, config kwargs) -- BASELINE.json
# configs[1..3] with SURVEY 8(d)'s seeds and schedules
CASES = {
    "config2": ((224, 192, 160), 1, 6.0,
                dict(nlevels=3, factors=[4, 2, 1], iters=[100, 75, 50], **{"lm.rejection": 1})),
    "config3_lm": ((224, 192, 224), 2, 8.0, dict(nlevels=4, factors=[8, 4, 2, 1], iters=[100, 100, 75, 50])),
    "config3_adam": ((224, 192, 224), 2, 8.0,
                     dict(nlevels=4, factors=[8, 4, 2, 1], iters=[100, 100, 75, 50], optimizer=1)),
    "config4": ((192, 192, 192), 1000, 6.0, dict(nlevels=1, factors=[1], iters=[100])),
}


def pair(name):
    shape, seed, wmax, _ = CASES[name]
    F, M, _ = O.synth_pair(shape, seed, num_blobs=12, warp_max=wmax)
    return F, M


def inputs_sha(F, M):
    return hashlib.sha256(np.ascontiguousarray(F).tobytes() + np.ascontiguousarray(M).tobytes()).hexdigest()


def sample_idx(shape):
    n = int(np.prod(shape))
    return np.sort(np.random.default_rng(12345).choice(n, NSAMPLE, replace=False))


def trace_array(tr):
    return np.array([(t.level, t.iter, t.r, t.lam, t.accepted, t.retries) for t in tr], dtype=np.float64)


def run(name):
    shape, seed, wmax, kw = CASES[name]
    F, M = pair(name)
    cfg = O.default_config(**kw)
    out = {"inputs_sha": np.array(inputs_sha(F, M)), "sample_idx": sample_idx(shape)}
    for var in ("fp64", "fp32"):
        t0 = time.time()
        if var == "fp32":
            with O.fp32_storage():
                rc, w, tr, jac = O.register(F, M, cfg)
        else:
            rc, w, tr, jac = O.register(F, M, cfg)
        assert rc == 0, (name, var, rc)
        flat = w.reshape(-1, 3)
        out[f"{var}_trace"] = trace_array(tr)
        out[f"{var}_warp_s"] = flat[out["sample_idx"]].astype(np.float32)  # the device stores fp32
        out[f"{var}_warp_norm"] = np.array(np.linalg.norm(w))
        out[f"{var}_jac"] = np.array(jac)
        print(f"{name} {var}: {len(tr)} iterations, {sum(int(t.retries) for t in tr)} retries, "
              f"final r {tr[-1].r:.8f}, {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), **out)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        run(name)
