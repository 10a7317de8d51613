"""Parity at BASELINE's full sizes (VERDICT r1 "next" #1).

Configs 2, 3 (LM and Adam) and 4 run through the product path on the B200
and are compared with the oracle's own runs of the same inputs, committed as
tests/golden/fullsize_*.npz by tests/golden/make_fullsize.py (the oracle
takes minutes per config on the host; the device seconds).  Every
comparison is made against two oracles:

  * fp32 storage -- the oracle with the device's fp32 storage points
    emulated (same algorithm, fp64 arithmetic): the trajectory the device
    should reproduce;
  * pure fp64    -- the north star's reference.

At these sizes the LM trajectory is chaotic: the fp32-storage oracle itself
leaves the fp64 one (loss > 1e-5 relative, then a different damping
decision) after a config-dependent number of iterations (the "storage
floor", measured from the fixtures themselves).  That span is one sample:
equally good fp32-storage trajectories spread widely around it
(tools/chaos_spread.py, profiles/r02/chaos_spread.json: the device on the
same pair with the last bit of the moving image flipped at a random half of
its voxels -- a change the size of one fp32 rounding -- leaves fp64 after
83-137 iterations on config 2 (storage oracle: 133), 82-135 on config 3 LM
(138), 58-100 on config 4 (58)).  So the fp64 bar is: loss within 1e-5 for
at least the shortest span of that study, accept/retry/lambda identical for
90% of the storage oracle's span, and a final warp no further from fp64
than the farthest perturbed run.  Against the fp32-storage oracle the bars
are stated per config below, with the measured values.

The final warps are compared on the fixtures' fixed sample of 2^15 voxels
(rel-L2 over the sample).  Inputs are regenerated with the oracle's
synth_pair and must hash to the fixture's inputs_sha.
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from golden.make_fullsize import CASES, inputs_sha, pair  # noqa: E402

pytestmark = pytest.mark.gpu

# Against the fp32-storage oracle, per config: loss tolerance, the number of
# leading iterations it must hold for (None = all), the number of leading
# iterations with identical accept/retry/lambda (None = all), and the
# sample warp rel-L2 bar (None: not stated, the chaotic tail dominates).
# Measured on the B200 (tools/fullsize_parity.py,
# profiles/r02/fullsize_parity.json): config 4 max loss 3.5e-7 over all
# 100, decisions all equal, warp 1.6e-4; config 2 loss <= 1e-5 for 185 of
# 225 accepted iterations, decisions equal for 186; config 3 LM loss
# <= 1e-6 for 82 of 325 iterations, decisions equal for 234.
# The device and this oracle are two fp64 implementations that differ only
# in operation order (K1b/K2 sum the shared taps of adjacent windows once,
# the oracle sums every window directly), and the chaotic trajectory grows
# those last-bit differences to 1e-5 within ~200 iterations -- later than
# fp32 storage itself does against fp64 (133 on config 2).  Until round 2's
# shared-tap sums (K1 -10%) K1b used the oracle's order and tracked config 2
# for all 225 iterations.
# Adam (config 3's baseline) is the most sensitive: its 28x24x28 first
# level leaves both oracles (1e-6 at iteration 59, 1e-5 at 63) although the
# first iterations agree to 5e-11 -- the oracles agree with each other to
# 167 because they share every fp64 operation order, the device does not
# (tools/diag_adam.py).  Its bars are stated separately.
STORAGE_BARS = {
    "config4": (1e-6, None, None, 1e-3),
    "config2": (1e-5, 170, 170, None),
    "config3_lm": (1e-6, 75, 210, None),
    "config3_adam": (1e-6, 50, None, None),
}
# Against the pure fp64 oracle, LM configs: (leading iterations within 1e-5,
# final-warp rel-L2 bar) = the shortest span and the farthest warp of the
# perturbation study (measured device: 133 / 0.0162, 107 / 0.0405,
# 58 / 0.0220); decisions as long as 90% of the storage oracle's.
FP64_SPAN = {"config2": (83, 0.040), "config3_lm": (82, 0.0563), "config4": (58, 0.0239)}
# Adam: (leading iterations within 1e-5, warp rel-L2 bar), measured 169 and
# 0.061 (its perturbed runs leave fp64 after 29-109 iterations: the study is
# no guide for it, so its earlier bars stay).
FP64_BARS = {"config3_adam": (55, 0.15)}


def first_divergence(a, b, tol):
    """(first iteration whose loss differs by > tol, first iteration whose
    level/iter/accepted/retries/lambda differ); len when none."""
    n = min(len(a), len(b))
    rel = np.abs(a[:n, 2] - b[:n, 2]) / np.abs(b[:n, 2])
    loss = next((k for k in range(n) if rel[k] > tol), n)
    dec = next((k for k in range(n) if not np.array_equal(a[k, [0, 1, 3, 4, 5]], b[k, [0, 1, 3, 4, 5]])), n)
    return loss, dec


def device_run(P, ctx, name, F, M):
    _, _, _, kw = CASES[name]
    cfg = P.reg_config(**kw)
    if kw["nlevels"] == 1:  # config 4: the bench's batch-engine path
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


@pytest.fixture(scope="module")
def P():
    import paper_2603_19371_b200 as P
    return P


@pytest.mark.parametrize("name", list(CASES))
def test_full_size_trajectory_vs_both_oracles(P, ctx, name):
    fx = np.load(os.path.join(HERE, "golden", f"fullsize_{name}.npz"))
    F, M = pair(name)
    assert inputs_sha(F, M) == str(fx["inputs_sha"]), "the oracle's synth_pair no longer makes the fixture's inputs"
    tr, warp = device_run(P, ctx, name, F, M)
    o32, o64 = fx["fp32_trace"], fx["fp64_trace"]
    assert len(tr) == len(o32) == len(o64)
    idx = fx["sample_idx"]
    w = warp.reshape(-1, 3)[idx]

    def wrel(ref):
        return np.linalg.norm(w - ref) / np.linalg.norm(ref)

    # fp32-storage oracle: the device's own trajectory
    tol, n_loss, n_dec, wbar = STORAGE_BARS[name]
    loss_k, dec_k = first_divergence(tr, o32, tol)
    assert loss_k >= (n_loss if n_loss is not None else len(tr)), (name, "loss vs storage oracle", loss_k)
    assert dec_k >= (n_dec if n_dec is not None else len(tr)), (name, "decisions vs storage oracle", dec_k)
    if wbar is not None:
        assert wrel(fx["fp32_warp_s"]) <= wbar, (name, wrel(fx["fp32_warp_s"]))
    # pure fp64 oracle: as long as fp32 storage itself allows
    loss_k, dec_k = first_divergence(tr, o64, 1e-5)
    if name in FP64_BARS:
        n_min, wbar64 = FP64_BARS[name]
        assert loss_k >= n_min and dec_k == len(tr), (name, loss_k, dec_k)
        assert wrel(fx["fp64_warp_s"]) <= wbar64, (name, wrel(fx["fp64_warp_s"]))
        return
    n_span, wbar64 = FP64_SPAN[name]
    _, floor_dec = first_divergence(o32, o64, 1e-5)
    assert loss_k >= n_span, (name, "loss vs fp64", loss_k, n_span)
    assert dec_k >= int(0.9 * floor_dec), (name, "decisions vs fp64", dec_k, floor_dec)
    assert wrel(fx["fp64_warp_s"]) <= wbar64, (name, wrel(fx["fp64_warp_s"]), wbar64)


def test_config5_decomposition_at_512_vs_oracle(P, ctx):
    """Config 5's path (GPU synth_pair of the config's kind: 96 blobs,
    displacement up to 8 at 512^3, z-slab group of 2 slabs with the
    interior / boundary overlap) against the fp32-storage oracle on the host
    for the first evaluation and 2 LM iterations: loss 1e-6, identical
    lambda, warp rel-L2 1e-6.  (The oracle cannot hold 1024^3 in host
    memory; 1024^3 itself is covered by P-invariance, test_gpu_parity.py.)"""
    import ctypes as C

    import oracle as O
    from paper_2603_19371_b200._lib import Dims, SynthSpec
    n, it = 512, 2
    shape = (n, n, n)
    F = np.empty(shape, np.float32)
    M = np.empty(shape, np.float32)
    spec = SynthSpec(Dims(n, n, n), 96, 0.0, 8.0, 0.01, 7)
    ctx.check(P.load().wlm_synth_pair(ctx.h, C.byref(spec), F.ctypes.data, M.ctypes.data, None, 0))
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[it])
    grp = P.SlabGroup(shape, 2, cfg=cfg, ctx=ctx)
    grp.load(F, M)
    grp.set_warp(None)
    grp.begin_level(0)
    grp.iterate(it)
    w, tr = grp.get_warp(), grp.trace()
    grp.close()
    L = O.lib()
    L.orc_set_threads(os.cpu_count() or 1)
    try:
        with O.fp32_storage():
            rc, u_o, _, tr_o = O.lm_run_level(F, M, np.zeros(shape + (3,)), O.default_config(
                nlevels=1, factors=[1], iters=[it]), it)
    finally:
        L.orc_set_threads(min(8, os.cpu_count() or 1))
    assert rc == 0 and len(tr) == len(tr_o) == it
    for a, b in zip(tr, tr_o):
        assert abs(a["r"] - b.r) <= 1e-6 * abs(b.r), (a["r"], b.r)
        assert a["lam"] == b.lam
    u_d = np.moveaxis(w.astype(np.float64), 0, -1)
    assert np.linalg.norm(u_d - u_o) / np.linalg.norm(u_o) <= 1e-6
