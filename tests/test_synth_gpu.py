"""The GPU synth_pair (csrc/synth.cu) against its closed-form recipe
("spot-check 10^5 random voxels against the CPU
formula"), and the bench's own GPU-generated 192^3 pair through the oracle.

The CPU restatement is tests/synth_formula.py (numpy): blob image, counter-
based SplitMix64 normals, separable fp32 smoothing of the noise field,
trilinear moving image.  The device uses __expf and fp32 sums, so the
comparison is to a few fp32 ulps of the unit range, not bitwise.
"""
import ctypes as C
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import synth_formula as SF  # noqa: E402

pytestmark = pytest.mark.gpu


def gpu_synth(P, ctx, shape, seed, blobs, wmax, noise):
    from paper_2603_19371_b200._lib import Dims, SynthSpec
    nz, ny, nx = shape
    F = np.empty(shape, np.float32)
    M = np.empty(shape, np.float32)
    U = np.empty((3,) + tuple(shape), np.float32)
    spec = SynthSpec(Dims(nx, ny, nz), blobs, 0.0, wmax, noise, seed)
    ctx.check(P.load().wlm_synth_pair(ctx.h, C.byref(spec), F.ctypes.data, M.ctypes.data, U.ctypes.data, 0))
    return F, M, U


@pytest.mark.parametrize("shape,seed,blobs,wmax", [((80, 72, 64), 1234, 12, 3.0), ((96, 96, 96), 1000, 12, 6.0)])
def test_gpu_synth_matches_formula_on_1e5_voxels(ctx, shape, seed, blobs, wmax):
    import paper_2603_19371_b200 as P
    noise = 0.01
    F, M, U = gpu_synth(P, ctx, shape, seed, blobs, wmax, noise)
    n = int(np.prod(shape))
    idx = np.random.default_rng(7).choice(n, 100000, replace=False)
    i64 = idx.astype(np.uint64)
    # fixed image: normalised blobs + N(0, noise^2) (stream 101)
    Fc = SF.clean_fixed(shape, seed, blobs)
    F_ref = (Fc.reshape(-1)[idx] + np.float32(noise) * SF.normal(seed, 101, i64)).astype(np.float32)
    assert np.abs(F.reshape(-1)[idx] - F_ref).max() < 2e-6
    # true warp: smoothed N(0, 1) field scaled to max |u| = warp_max (first draw)
    U_ref = SF.true_warp(shape, seed, wmax)
    assert abs(np.abs(U).max() - wmax) < 1e-5 * wmax
    assert np.abs(U.reshape(3, -1)[:, idx] - U_ref.reshape(3, -1)[:, idx]).max() < 2e-5 * wmax
    # moving image: clean F at x + u_true (trilinear, fp64 lerps) + noise (stream 102)
    M_ref = SF.sample_exact(Fc, U, idx) + np.float32(noise) * SF.normal(seed, 102, i64)
    assert np.abs(M.reshape(-1)[idx] - M_ref).max() < 5e-6


def test_bench_pair_through_the_oracle(ctx):
    """The bench's first config-4 pair (GPU synth_pair, seed 1000, 192^3,
    warp_max 6) -- the inputs the benchmark actually times -- for 10 LM
    iterations against the fp32-storage oracle (loss 1e-6, identical
    decisions and lambda) and the fp64 oracle (loss 1e-5)."""
    import oracle as O
    import paper_2603_19371_b200 as P
    shape = (192, 192, 192)
    F, M, _ = gpu_synth(P, ctx, shape, 1000, 12, 6.0, 0.01)
    it = 10
    eng = P.Engine(shape, pairs=1, cfg=P.reg_config(nlevels=1, factors=[1], iters=[it]), ctx=ctx)
    eng.load(F[None], M[None])
    eng.set_warp(None)
    eng.begin_level(0)
    eng.iterate(it)
    tr = eng.trace(0)
    eng.close()
    cfg_o = O.default_config(nlevels=1, factors=[1], iters=[it])
    for storage, tol in (("fp32", 1e-6), ("fp64", 1e-5)):
        if storage == "fp32":
            with O.fp32_storage():
                rc, _, _, tr_o = O.lm_run_level(F, M, np.zeros(shape + (3,)), cfg_o, it)
        else:
            rc, _, _, tr_o = O.lm_run_level(F, M, np.zeros(shape + (3,)), cfg_o, it)
        assert rc == 0 and len(tr_o) == len(tr) == it
        for a, b in zip(tr, tr_o):
            assert abs(a["r"] - b.r) <= tol * abs(b.r), (storage, a["r"], b.r)
            assert a["lam"] == b.lam and a["accepted"] == b.accepted
