"""GPU parity tests: the sm_100a path (through the C-ABI) against the fp64
oracle on identical seeded inputs.

Tolerances (stated once):
  * field ops in fp32 vs the fp64 reference: max abs error <= 1e-5 * scale
    (inputs O(1)), exact where the SPEC says exact;
  * LNCC residual r: rel <= 1e-5 (north star); gradient rel-L2 <= 1e-4;
  * LM runs: per-iteration loss rel <= 1e-5, identical accept/reject
    sequence, final warp rel-L2 <= 1e-4, lambda bit-identical.
"""
import math

import numpy as np
import pytest

import oracle as O
from conftest import rel, smooth_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2603_19371_b200 as P
    return P


def soa(u):
    """(nz,ny,nx,3) AoS -> (3,nz,ny,nx) SoA float32."""
    return np.ascontiguousarray(np.moveaxis(u, -1, 0), dtype=np.float32)


def aos(u):
    return np.moveaxis(np.asarray(u, np.float64), 0, -1)


# ------------------------------------------------------------ field ops ----
# The field-module mirrors keep the caller's fp64 data and run the
# reference's expressions in its operation order on the device (field64.cu),
# so they are compared with the UNMODIFIED reference's own outputs
# (tests/golden/field_ref.npz, tests/golden/make_golden.py) bit for bit.
def same_bits(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def test_compose_vs_reference(P, ctx, golden):
    for name in ("c6", "c876"):
        u, v, eps = golden[f"{name}_u"], golden[f"{name}_v"], float(golden[f"{name}_eps"])
        assert same_bits(P.compose_warp(u, v, eps, ctx=ctx), golden[f"{name}_out"]), name
    v = np.random.default_rng(0).normal(size=(6, 6, 6, 3))
    assert np.array_equal(P.compose_warp(np.zeros_like(v), v, 0.5, ctx=ctx), 0.5 * v)
    c = np.full((5, 6, 7, 3), 1.25)
    assert np.array_equal(P.compose_warp(c, np.zeros_like(c), 0.3, ctx=ctx), c)
    with pytest.raises(P.DimensionMismatch):
        P.compose_warp(np.zeros((4, 4, 4, 3)), np.zeros((4, 4, 5, 3)), 0.1, ctx=ctx)


@pytest.mark.parametrize("key", ["1p0", "0p5", "2p3"])
def test_smooth_vs_reference(P, ctx, golden, key):
    sig = float(key.replace("p", "."))
    for kind in ("field", "vol"):
        out = P.gaussian_smooth(golden[f"sm{key}_{kind}_in"], sig, ctx=ctx)
        assert same_bits(out, golden[f"sm{key}_{kind}_out"]), kind
    c = np.full((7, 8, 9), 2.5)
    assert np.abs(P.gaussian_smooth(c, 1.0, ctx=ctx) - 2.5).max() < 1e-15  # constants preserved


def test_smooth_any_sigma_matches_oracle(P, ctx):
    """gaussian_smooth for any sigma > 0 (radius ceil(3 sigma), field.cpp:206),
    including sigma > 2 (radius 7 and 19 here) and an n == 1 axis."""
    rng = np.random.default_rng(11)
    for shape, sig in (((9, 10, 11), 2.5), ((1, 12, 40), 6.2), ((8, 9, 10), 0.2)):
        a = rng.normal(size=shape + (3,))
        assert same_bits(P.gaussian_smooth(a, sig, ctx=ctx), O.gaussian_smooth(a, sig)), (shape, sig)


def test_max_normalize_jacobian(P, ctx, golden):
    u = golden["jac_u"]
    assert P.max_abs_component(u, ctx=ctx) == float(golden["max_out"])
    assert P.normalize_step(u, ctx=ctx) == float(golden["norm_out"])
    assert P.jacobian_det_min(u, ctx=ctx) == float(golden["jac_out"])
    assert P.jacobian_det_min(golden["jac2_u"], ctx=ctx) == float(golden["jac2_out"])
    with pytest.raises(P.InvalidArgument):
        P.normalize_step(u, P.StepScale(0.6), ctx=ctx)  # field.cpp:151-153
    with pytest.raises(P.InvalidArgument):
        P.jacobian_det_min(np.zeros((1, 4, 4, 3)), ctx=ctx)  # field.cpp:174-176
    z = np.zeros((5, 5, 5, 3))
    assert P.jacobian_det_min(z, ctx=ctx) == 1.0
    r = z.copy(); r[..., 0] = 0.1 * np.arange(5)
    assert P.jacobian_det_min(r, ctx=ctx) == 1.1000000000000001  # SPEC.md:82, the reference's own value


def test_sample_trilinear_grad_points_vs_reference(P, ctx, golden):
    """Per-point sample_trilinear_grad (field.hpp:90) at the golden points:
    knots, borders, outside, NaN/inf coordinates."""
    val, grad = P.sample_trilinear_grad(golden["sample_vol"], golden["sample_pts"], ctx=ctx)
    ref_v, ref_g = golden["sample_val"], golden["sample_grad"]
    fin = np.isfinite(ref_v)
    assert np.array_equal(np.isnan(val), ~fin)
    assert same_bits(val[fin], ref_v[fin]) and same_bits(grad[fin], ref_g[fin])
    assert np.array_equal(P.sample_trilinear(golden["sample_vol"], golden["sample_pts"][:5], ctx=ctx), val[:5])


def test_warp_volume_vs_reference(P, ctx, golden):
    rng = np.random.default_rng(5)
    M = rng.normal(size=(11, 12, 13))
    u = smooth_field((11, 12, 13), 1, amp=3.0)
    u[0, 0, 0] = (0.0, 0.0, 0.0)  # exact knot
    u[1, 1, 1] = (-1e-9, 0, 0)    # just below a knot: backward difference
    Mw, gM = P.warp_volume(M, u, ctx=ctx)
    kind = "reference" if O.have_ref() else "port"  # the port is bit-identical (test_oracle.py)
    Mo, go = O.warp_volume(M, u, kind=kind)
    assert same_bits(Mw, Mo) and same_bits(gM, go)


def test_sample_field_and_pyramid(P, ctx):
    u = smooth_field((8, 9, 10), 2, amp=1.0)
    pts = np.random.default_rng(3).uniform(-2, 11, size=(500, 3))
    got = P.sample_field(u, pts, ctx=ctx)
    ref = np.array([_sample3(u, p) for p in pts])
    assert same_bits(got, ref)
    vol = np.random.default_rng(4).uniform(size=(20, 18, 17))
    for f in (2, 3, 4):
        d = P.downsample(vol, f, ctx=ctx)
        assert d.shape == O.level_dims(vol.shape, f)
        assert same_bits(d, O.downsample(vol, f))
    up = P.upsample_warp(u, (16, 18, 20), 2.0, ctx=ctx)
    assert same_bits(up, O.upsample_warp(u, (16, 18, 20), 2.0))


def _sample3(u, p):
    out = np.empty(3)
    import ctypes as C
    uu = np.ascontiguousarray(u)
    O.lib().orc_sample_field(O._p(uu), O.dims_of(uu), float(p[0]), float(p[1]), float(p[2]), O._p(out))
    return out


def test_all_finite(P, ctx):
    a = np.zeros((4, 4, 4, 3))
    assert P.all_finite(a, ctx=ctx)
    a[1, 2, 3, 1] = np.nan
    assert not P.all_finite(a, ctx=ctx)
    b = np.zeros((4, 4, 4)); b[0, 0, 0] = np.inf
    assert not P.all_finite(b, ctx=ctx)


# --------------------------------------------------------------- LNCC ----
def _pair(shape, seed, warp_max=2.0, noise=0.01):
    F, M, _ = O.synth_pair(shape, seed, num_blobs=8, warp_max=warp_max, noise_sigma=noise)
    return F.astype(np.float64), M.astype(np.float64)


@pytest.mark.parametrize("shape,offset", [((24, 20, 28), 0.0), ((33, 17, 21), 0.0), ((24, 24, 24), 10.0)])
def test_residual_lncc_vs_oracle(P, ctx, shape, offset):
    F, M = _pair(shape, 11)
    F, M = F + offset, M + offset
    F = F.astype(np.float32).astype(np.float64)
    M = M.astype(np.float32).astype(np.float64)
    u = smooth_field(shape, 6, amp=1.5).astype(np.float32).astype(np.float64)
    rep = P.residual_lncc(F, M, u, ctx=ctx)
    r, g, ln = O.residual_lncc(F, M, u)
    assert abs(rep.r - r) / r < 1e-5
    assert abs(rep.loss_raw - ln) < 1e-5
    assert rel(rep.g, g) < 1e-4, rel(rep.g, g)


def test_lncc_kats_gpu(P, ctx):
    F, _ = _pair((16, 16, 16), 5, warp_max=0.0, noise=0.05)
    F32 = F.astype(np.float32).astype(np.float64)
    z = np.zeros(F.shape + (3,))
    rep = P.residual_lncc(F32, (2 * F32 + 3).astype(np.float32).astype(np.float64), z, ctx=ctx)
    assert abs(rep.loss_raw - 1.0) < 1e-5 and abs(rep.r) < 1e-5
    rep = P.residual_lncc(np.full((10, 10, 10), 0.7), F32[:10, :10, :10], z[:10, :10, :10], ctx=ctx)
    assert rep.loss_raw == 0.0 and rep.r == 1.0 and not rep.g.any()
    with pytest.raises(P.InvalidArgument):
        P.residual_lncc(F32[:4], F32[:4], z[:4], ctx=ctx)


def test_lm_step_pointwise_gpu(P, ctx):
    g = np.zeros((2, 2, 2, 3)); g[0, 0, 0] = (1, 0, 0)
    out = P.lm_step_pointwise(2.0, g, 1.0, ctx=ctx)
    assert np.array_equal(out[0, 0, 0], [-1.0, 0.0, 0.0]) and not out[1:].any()
    gg = np.random.default_rng(2).normal(size=(5, 6, 7, 3))
    assert same_bits(P.lm_step_pointwise(0.3, gg, 0.01, ctx=ctx), O.lm_step_pointwise(0.3, gg, 0.01))


# ------------------------------------------------------------ LM engine ----
def run_engine(P, ctx, F, M, cfg, iters, u0=None, pairs=1):
    eng = P.Engine(F.shape[-3:], pairs=pairs, cfg=cfg, ctx=ctx)
    Fb = np.broadcast_to(F, (pairs,) + F.shape[-3:]) if F.ndim == 3 else F
    Mb = np.broadcast_to(M, (pairs,) + M.shape[-3:]) if M.ndim == 3 else M
    eng.load(np.ascontiguousarray(Fb, np.float32), np.ascontiguousarray(Mb, np.float32))
    eng.set_warp(u0)
    eng.begin_level(0)
    eng.iterate(iters)
    warp = eng.get_warp()
    traces = [eng.trace(p) for p in range(pairs)]
    states = [eng.state(p) for p in range(pairs)]
    eng.close()
    return warp, traces, states


def compare_runs(tr_gpu, tr_orc, warp_gpu, warp_orc, loss_tol=1e-5, warp_tol=1e-4, first_n=None):
    """Per-iteration loss within loss_tol (for the first first_n iterations
    when given), identical accept/retry sequence and lambda (bit-exact: the
    device state machine is the oracle's fp64 arithmetic), final warp rel-L2."""
    assert len(tr_gpu) == len(tr_orc)
    for k, (a, b) in enumerate(zip(tr_gpu, tr_orc)):
        ga = a if isinstance(a, dict) else dict(r=a.r, accepted=a.accepted, retries=a.retries,
                                               lam=a.lam, iter=a.iter)
        if first_n is None or k < first_n:
            assert abs(ga["r"] - b.r) <= loss_tol * abs(b.r), (k, ga["r"], b.r)
        assert ga["accepted"] == b.accepted and ga["retries"] == b.retries, k
        assert ga["lam"] == b.lam, (k, ga["lam"], b.lam)
    if warp_tol is not None:
        assert rel(warp_gpu, warp_orc) <= warp_tol, rel(warp_gpu, warp_orc)


def oracle_level(F, M, cfg_o, iters, storage):
    """lm_run_level with the pure fp64 oracle ('fp64') or with the device's
    fp32 storage points emulated ('fp32')."""
    if storage == "fp32":
        with O.fp32_storage():
            return O.lm_run_level(F, M, np.zeros(F.shape + (3,)), cfg_o, iters)
    return O.lm_run_level(F, M, np.zeros(F.shape + (3,)), cfg_o, iters)


# Parity bar:
#  * vs the fp32-storage oracle (same fp32 storage points, fp64 arithmetic):
#    loss <= 1e-6 relative at every iteration, identical accept/reject and
#    lambda, final warp rel-L2 <= 1e-5 -- measured 1e-14..2e-8 / 0..1.4e-7;
#  * vs the pure fp64 reference oracle: the north-star bar (loss <= 1e-5,
#    identical accept/reject, warp rel-L2 <= 1e-4) on single-level runs --
#    measured <= 2.2e-8 / 1.2e-6 -- and, where fp32 storage itself is chaotic
#    (tiny coarse pyramid levels, tools/floor_experiment.py), the first 20
#    iterations plus the full accept/reject sequence.
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_config1_64cubed_100_iterations(P, ctx, seed):
    """Config 1 (BASELINE.json): 64^3, one level, LNCC, 100 LM iterations
    (seed 0 is the config's; 1 and 2 are the trajectories the precision study
    found most sensitive)."""
    F, M, _ = O.synth_pair((64, 64, 64), seed, num_blobs=12, warp_max=3.0)
    cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[100])
    cfg_o = O.default_config(nlevels=1, factors=[1], iters=[100])
    warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, 100)
    # seed 1's late, oscillating iterations amplify 1e-8 differences: its final
    # warp sits 2e-5 from the storage oracle (loss and decisions stay tight)
    wt32 = 1e-5 if seed == 0 else 1e-4
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, wt32)):
        rc, u_o, st, tr_o = oracle_level(F, M, cfg_o, 100, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)


def test_rejection_sequence_matches(P, ctx):
    """LM + capped rejection: identical accept/reject sequence (north star)."""
    F, M, _ = O.synth_pair((32, 36, 40), 3, num_blobs=10, warp_max=3.0)
    kw = dict(nlevels=1, factors=[1], iters=[40])
    cfg_p = P.reg_config(**kw, **{"lm.rejection": 1, "lm.tau": 0.2})
    cfg_o = O.default_config(**kw, **{"lm.rejection": 1, "lm.tau": 0.2})
    warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, 40)
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
        rc, u_o, st, tr_o = oracle_level(F, M, cfg_o, 40, storage)
        assert rc == 0
        assert sum(t.retries for t in tr_o) > 0, "test should exercise rejections"
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)


def test_scripted_losses_lambda_trajectory(P, ctx):
    """SPEC.md:290 scripted-residual harness on the device state machine."""
    F, M, _ = O.synth_pair((16, 16, 16), 1, warp_max=1.0)
    losses = np.r_[1.0, 0.9, np.full(11, 5.0), 0.8, 0.7, 0.75, 0.6]
    cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[6], **{"lm.rejection": 1})
    eng = P.Engine((16, 16, 16), 1, cfg_p, ctx=ctx)
    eng.load(F[None], M[None])
    eng.set_warp(None)
    eng.script_losses(losses[None])
    eng.begin_level(0)
    eng.iterate(6)
    tr = eng.trace(0)
    lam, dec, st = O.lm_replay(losses, 6, O.lm_config(rejection=1))
    acc_lams = [l for l, d in zip(lam, dec) if d == 0]
    assert [t["lam"] for t in tr] == acc_lams
    assert [t["retries"] for t in tr] == [0, 0, 10, 0, 0, 0]
    assert tr[2]["accepted"] == 0  # forced after 10 retries
    assert eng.state(0)["lam"] == st.lam
    eng.close()


def same_trace(a, b):
    """Row-wise equality with NaN == NaN (jac_det_min is NaN when not logged)."""
    if isinstance(a, list) and a and isinstance(a[0], list):
        return len(a) == len(b) and all(same_trace(x, y) for x, y in zip(a, b))
    return len(a) == len(b) and all(
        all((x[k] == y[k]) or (x[k] != x[k] and y[k] != y[k]) for k in x) for x, y in zip(a, b))


@pytest.mark.parametrize("shape", [(1, 9, 10), (7, 1, 6), (5, 6, 1), (2, 3, 4), (3, 17, 33), (5, 6, 7),
                                   (6, 13, 21), (9, 10, 37)])
def test_degenerate_and_ragged_dims_match_oracle(P, ctx, shape):
    """n == 1 axes (resolve_axis collapse, field.cpp:21-24; smoothing skipped,
    :220), two-voxel axes, and widths that are not multiples of 4 (K4's
    register-staged path instead of TMA): the ops and a rejection-on LM run
    against the fp32-storage oracle.  LNCC needs every dim > 2 radius
    (SPEC.md:138); thinner volumes run MSE."""
    rng = np.random.default_rng(sum(shape))
    F = O.gaussian_smooth(rng.normal(size=shape), 1.0).astype(np.float32)
    M = O.gaussian_smooth(rng.normal(size=shape), 1.0).astype(np.float32)
    F64, M64 = F.astype(np.float64), M.astype(np.float64)
    u = smooth_field(shape, 7, sigma=1.0, amp=1.5).astype(np.float32).astype(np.float64)
    v = smooth_field(shape, 8, sigma=1.0, amp=1.0).astype(np.float32).astype(np.float64)
    assert np.abs(P.compose_warp(u, v, 0.3, ctx=ctx) - O.compose_warp(u, v, 0.3)).max() < 2e-5
    for sig in (1.0, 0.5):
        assert np.abs(P.gaussian_smooth(u, sig, ctx=ctx) - O.gaussian_smooth(u, sig)).max() < 2e-6
    lncc = min(shape) > 4
    if lncc:
        rep = P.residual_lncc(F64, M64, u, ctx=ctx)
        r_o, g_o, _ = O.residual_lncc(F64, M64, u)
    else:
        with pytest.raises(P.InvalidArgument):
            P.residual_lncc(F64, M64, u, ctx=ctx)
        rep = P.residual_mse(F64, M64, u, ctx=ctx)
        r_o, g_o = O.residual_mse(F64, M64, u)
    assert abs(rep.r - r_o) <= 1e-5 * abs(r_o)
    assert rel(rep.g, g_o) < 1e-4, rel(rep.g, g_o)
    kw = dict(nlevels=1, factors=[1], iters=[12], metric=0 if lncc else 1)
    cfg_p = P.reg_config(**kw, **{"lm.rejection": 1, "lm.tau": 0.5})
    cfg_o = O.default_config(**kw, **{"lm.rejection": 1, "lm.tau": 0.5})
    warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, 12)
    rc, u_o, _, tr_o = oracle_level(F, M, cfg_o, 12, "fp32")
    assert rc == 0
    compare_runs(tr, tr_o, aos(warp[0]), u_o, 1e-6, 1e-5)


@pytest.mark.parametrize("rejection", [0, 1])
def test_pair_groups_do_not_change_results(P, ctx, rejection):
    """Pair-group streams (the default: 2) vs one chain: bit-identical warps
    and traces, with an odd pair count (groups of 2 and 1, or 1, 1, 1), with
    rejection off (graph streams) and on (one WHILE graph per group)."""
    shape = (24, 28, 32)
    Fs, Ms = zip(*[O.synth_pair(shape, 300 + s, num_blobs=10, warp_max=3.0)[:2] for s in range(3)])
    F, M = np.stack(Fs), np.stack(Ms)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[40], **{"lm.rejection": rejection, "lm.tau": 0.2})
    out = {}
    for groups in (1, 2, 3):
        eng = P.Engine(shape, pairs=3, cfg=cfg, ctx=ctx)
        eng.set_pair_groups(groups)
        eng.load(F, M)
        eng.set_warp(None)
        eng.begin_level(0)
        eng.iterate(25)
        eng.iterate(15)
        out[groups] = (eng.get_warp(), [eng.trace(p) for p in range(3)])
        eng.close()
    for groups in (2, 3):
        assert np.array_equal(out[1][0], out[groups][0])
        assert same_trace(out[1][1], out[groups][1]) and len(out[groups][1][2]) == 40
    if rejection:
        assert sum(t["retries"] for tr in out[2][1] for t in tr) > 0, "should exercise rejections"
    with pytest.raises(P.InvalidArgument):
        P.Engine(shape, pairs=1, cfg=cfg, ctx=ctx).set_pair_groups(5)


def test_batch_pairs_are_independent_and_deterministic(P, ctx):
    shape = (24, 28, 32)
    Fs, Ms = [], []
    for s in range(3):
        F, M, _ = O.synth_pair(shape, 100 + s, num_blobs=6, warp_max=2.0)
        Fs.append(F); Ms.append(M)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[15])
    wb, trb, _ = run_engine(P, ctx, np.stack(Fs), np.stack(Ms), cfg, 15, pairs=3)
    wb2, trb2, _ = run_engine(P, ctx, np.stack(Fs), np.stack(Ms), cfg, 15, pairs=3)
    assert np.array_equal(wb, wb2) and same_trace(trb, trb2)  # bit-identical reruns
    for s in range(3):
        w1, (t1,), _ = run_engine(P, ctx, Fs[s], Ms[s], cfg, 15)
        assert np.array_equal(w1[0], wb[s]) and same_trace(t1, trb[s])


def test_adam_and_gd_paths(P, ctx):
    F, M, _ = O.synth_pair((24, 24, 24), 8, num_blobs=6, warp_max=2.0)
    for opt, extra in ((P.OPT_ADAM, {}), (P.OPT_GD, {"gd_lr": 2.0})):
        cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[20], optimizer=opt, **extra)
        cfg_o = O.default_config(nlevels=1, factors=[1], iters=[20], optimizer=opt, **extra)
        warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, 20)
        for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
            rc, u_o, _, tr_o = oracle_level(F, M, cfg_o, 20, storage)
            for a, b in zip(tr, tr_o):
                assert abs(a["r"] - b.r) <= lt * b.r
            assert rel(aos(warp[0]), u_o) < wt


def test_jacobian_logged_positive(P, ctx):
    F, M, _ = O.synth_pair((20, 20, 20), 4, warp_max=2.0)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[10], log_jacobian=1)
    _, (tr,), _ = run_engine(P, ctx, F, M, cfg, 10)
    cfg_o = O.default_config(nlevels=1, factors=[1], iters=[10], log_jacobian=1)
    _, _, _, tr_o = O.lm_run_level(F, M, np.zeros((20, 20, 20, 3)), cfg_o, 10)
    for a, b in zip(tr, tr_o):
        assert a["jac_det_min"] > 0
        assert abs(a["jac_det_min"] - b.jac_det_min) < 1e-4


def test_register_pyramid_vs_oracle(P, ctx):
    """Config-2-shaped pyramid (scaled down): levels, warp inheritance,
    lambda carry, rejection on."""
    F, M, _ = O.synth_pair((40, 48, 56), 1, num_blobs=10, warp_max=4.0)
    kw = dict(nlevels=3, factors=[4, 2, 1], iters=[30, 20, 10])
    res = P.register(F, M, P.reg_config(**kw, **{"lm.rejection": 1}), ctx=ctx)
    cfg_o = O.default_config(**kw, **{"lm.rejection": 1})
    # fp64 reference: the 10x12x14 first level is floor-limited (the oracle
    # against itself with fp32 warps reaches 8e-6 by iteration 27), so the
    # loss bar holds for the first 20 iterations and the accept/reject
    # sequence and lambda for all 60.
    rc, w_o, tr_o, jac_o = O.register(F, M, cfg_o)
    assert rc == 0 and len(res.loss_trace) == len(tr_o) == 60
    for a, b in zip(res.loss_trace, tr_o):
        assert (a.level, a.iter) == (b.level, b.iter)
    compare_runs(res.loss_trace, tr_o, res.final_warp, w_o, 1e-5, None, first_n=20)
    # fp32-storage oracle: the whole pyramid, tight
    with O.fp32_storage():
        rc, w_s, tr_s, jac_s = O.register(F, M, cfg_o)
    compare_runs(res.loss_trace, tr_s, res.final_warp, w_s, 1e-6, 1e-5)
    assert res.jac_det_min_final == pytest.approx(jac_s, abs=1e-4)
    assert res.peak_device_bytes > 0


def test_nonfinite_input_aborts(P, ctx):
    F, M, _ = O.synth_pair((16, 16, 16), 1, warp_max=1.0)
    M = M.copy(); M[3, 3, 3] = np.nan
    with pytest.raises(P.NonFiniteLoss):
        P.register(F, M, P.reg_config(nlevels=1, factors=[1], iters=[3]), ctx=ctx)


def test_cpp_adapter_runs_on_gpu(tmp_path):
    """A reference-style C++ caller (tests/cpp/adapter_demo.cpp) through the
    ABI: compose_warp KAT, normalize_step, dim-mismatch exception."""
    import subprocess
    from test_abi import build_adapter_demo
    exe = build_adapter_demo(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


# ------------------------------------------------------- z-slab groups ----
def run_slabs(P, ctx, F, M, cfg, iters, nslabs, want_fused=None):
    grp = P.SlabGroup(F.shape, nslabs, cfg=cfg, ctx=ctx)
    if want_fused is not None:
        assert grp.fused_halos() == want_fused, (nslabs, grp.fused_halos(), want_fused)
    grp.load(F, M)
    grp.set_warp(None)
    grp.begin_level(0)
    grp.iterate(iters)
    out = grp.get_warp(), grp.trace(), grp.state()
    grp.close()
    return out


@pytest.mark.parametrize("extra", [{}, {"lm.rejection": 1, "lm.tau": 0.2, "log_jacobian": 1},
                                   {"optimizer": 1}, {"sigma_update": 2.0, "sigma_warp": 1.6},
                                   {"low_memory": 1, "lm.rejection": 1, "lm.tau": 0.2}])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_slab_group_is_bit_identical_to_single_domain(P, ctx, extra, fused, monkeypatch):
    """Config 5 decomposition: 1, 2, 3 and 5 z-slabs (uneven splits) give the
    single-domain engine's losses, decisions, lambda and warp bit for bit,
    with the producers' fused halo stores (default) and with the copy
    exchange (WLM_SLAB_FUSED=0)."""
    monkeypatch.setenv("WLM_SLAB_FUSED", fused)
    F, M, _ = O.synth_pair((20, 24, 28), 21, num_blobs=8, warp_max=2.5)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[12], **extra)
    w1, (t1,), (s1,) = run_engine(P, ctx, F, M, cfg, 12)
    # wide kernels (radius 6 / 5) need 6 halo planes: at most 3 slabs of 20
    # fused kinds: g unless Adam (its step is produced by k_adam), dU_s, the
    # warp and A/B/E; none with one slab or with WLM_SLAB_FUSED=0
    mask = 0b1111 if extra.get("optimizer", 0) != 1 else 0b1110
    for ns in ((1, 2, 3) if "sigma_warp" in extra else (1, 2, 3, 5)):
        w, t, s = run_slabs(P, ctx, F, M, cfg, 12, ns, want_fused=mask if fused == "1" and ns > 1 else 0)
        assert same_trace(t, t1), ns
        assert np.array_equal(w, w1[0]), (ns, float(np.abs(w - w1[0]).max()))
        assert s["lam"] == s1["lam"] and s["r"] == s1["r"]


def test_slab_group_rejects_thin_slabs(P, ctx):
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[1])
    with pytest.raises(P.InvalidArgument):
        P.SlabGroup((12, 16, 16), 4, cfg=cfg, ctx=ctx)


@pytest.mark.parametrize("extra", [{}, {"lm.rejection": 1, "lm.tau": 0.2, "log_jacobian": 1},
                                   {"metric": 2, "mi_bins": 16}])
def test_nccl_rank_slab_world1_matches_engine(P, ctx, extra):
    """The one-process-per-GPU transport on a real NCCL communicator of one
    rank: plane-sum and max all-reduces, foreign-plane zeroing and the eager
    attempt loop (with rejection) give the engine's result bit for bit."""
    from paper_2603_19371_b200 import slabs
    F, M, _ = O.synth_pair((20, 24, 28), 22, num_blobs=8, warp_max=2.5)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[10], **extra)
    w1, (t1,), (s1,) = run_engine(P, ctx, F, M, cfg, 10)
    grp = slabs.RankSlab(F.shape, 0, 1, slabs.nccl_unique_id(), cfg=cfg, ctx=ctx)
    grp.load(F, M)
    grp.set_warp(None)
    grp.begin_level(0)
    grp.iterate(10)
    assert grp.owned() == (0, F.shape[0])
    w, t = grp.get_local_warp(), grp.trace()
    grp.close()
    assert same_trace(t, t1)
    assert np.array_equal(w, w1[0])


# ------------------------------------------------------------------- MSE ----
def test_residual_mse_vs_oracle(P, ctx):
    F, M = _pair((20, 22, 24), 12)
    F = F.astype(np.float32).astype(np.float64)
    M = M.astype(np.float32).astype(np.float64)
    u = smooth_field(F.shape, 7, amp=1.2).astype(np.float32).astype(np.float64)
    rep = P.residual_mse(F, M, u, ctx=ctx)
    r, g = O.residual_mse(F, M, u)
    assert abs(rep.r - r) <= 1e-12 * r and rep.loss_raw == rep.r
    assert rel(rep.g, g) < 1e-6, rel(rep.g, g)
    z = np.zeros(F.shape + (3,))
    assert P.residual_mse(F, F, z, ctx=ctx).r == 0.0
    assert P.residual_mse(np.zeros_like(F), np.ones_like(F), z, ctx=ctx).r == 1.0


def test_mse_engine_vs_oracle(P, ctx):
    """MetricConfig.kind = mse through the device engine (K1a + MSE partials,
    pointwise MSE gradient, same step / smoothing / compose kernels)."""
    F, M, _ = O.synth_pair((32, 36, 40), 6, num_blobs=10, warp_max=3.0)
    kw = dict(nlevels=1, factors=[1], iters=[30], metric=1)
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 30)
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
        rc, u_o, st, tr_o = oracle_level(F, M, O.default_config(**kw), 30, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    assert all(t["r"] == t["loss_raw"] for t in tr)


def test_mse_slab_group_bit_identical(P, ctx):
    F, M, _ = O.synth_pair((20, 24, 28), 23, num_blobs=8, warp_max=2.5)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[10], metric=1)
    w1, (t1,), _ = run_engine(P, ctx, F, M, cfg, 10)
    w, t, _ = run_slabs(P, ctx, F, M, cfg, 10, 3)
    assert same_trace(t, t1) and np.array_equal(w, w1[0])


# ---------------------------------------------------------------- Demons ----
def test_demons_step_mirror_bitwise(P, ctx):
    rng = np.random.default_rng(5)
    r = rng.normal(size=(6, 7, 8))
    n = rng.normal(size=(6, 7, 8, 3))
    r[0, 0, 0] = 0.0; n[0, 0, 0] = 0.0  # zero denominator -> 0
    for alpha in (0.5, 1.0):
        assert np.array_equal(P.demons_step_mse(r, n, alpha, ctx=ctx), O.demons_step_mse(r, n, alpha))
    out = P.demons_step_mse(np.ones((1, 1, 1)), np.array([[[[2.0, 0, 0]]]]), 1.0, ctx=ctx)
    assert np.allclose(out[0, 0, 0], [0.4, 0, 0], rtol=0, atol=1e-15)


def test_demons_engine_vs_oracle(P, ctx):
    F, M, _ = O.synth_pair((24, 28, 32), 9, num_blobs=8, warp_max=2.5)
    kw = dict(nlevels=1, factors=[1], iters=[20], metric=1, optimizer=3, demons_alpha=1.0)
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 20)
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
        rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 20, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    with pytest.raises(P.InvalidArgument):  # Demons needs the MSE per-voxel residual
        P.Engine((8, 8, 8), 1, P.reg_config(optimizer=3), ctx=ctx)


# -------------------------------------------------------------- tiled LM ----
def test_tiled_lm_mirror_bitwise(P, ctx):
    rng = np.random.default_rng(9)
    for shape, k in (((6, 6, 6), 3), ((7, 5, 9), 2), ((9, 8, 7), 4), ((5, 6, 7), 1)):
        g = rng.normal(size=shape + (3,))
        assert np.array_equal(P.lm_step_tiled(0.3, g, 0.2, k, ctx=ctx), O.lm_step_tiled(0.3, g, 0.2, k))


@pytest.mark.parametrize("k", [2, 3])
def test_tiled_lm_engine_vs_oracle(P, ctx, k):
    F, M, _ = O.synth_pair((24, 28, 32), 14, num_blobs=8, warp_max=2.5)
    kw = dict(nlevels=1, factors=[1], iters=[20], **{"lm.tile_size": k})
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 20)
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
        rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 20, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    # z-slabs: tile-aligned boundaries + step matrices of the halo tiles
    for ns in (2, 3):
        w, t, _ = run_slabs(P, ctx, F, M, P.reg_config(**kw), 20, ns)
        assert same_trace(t, tr) and np.array_equal(w, warp[0]), (k, ns)


# -------------------------------------------------------------------- MI ----
def test_residual_mi_vs_oracle(P, ctx):
    F, M = _pair((20, 22, 24), 13)
    F = F.astype(np.float32).astype(np.float64)
    M = M.astype(np.float32).astype(np.float64)
    u = smooth_field(F.shape, 8, amp=1.2).astype(np.float32).astype(np.float64)
    for bins, sigma in ((32, 1.0), (16, 0.5)):
        rep = P.residual_mi(F, M, u, bins=bins, sigma=sigma, ctx=ctx)
        r, g, mi = O.residual_mi(F, M, u, bins=bins, sigma=sigma)
        assert abs(rep.r - r) <= 1e-9 * r and abs(rep.loss_raw - mi) <= 1e-9
        assert rel(rep.g, g) < 1e-6, rel(rep.g, g)


def test_mi_engine_vs_oracle(P, ctx):
    F, M, _ = O.synth_pair((24, 28, 32), 15, num_blobs=10, warp_max=2.5)
    kw = dict(nlevels=1, factors=[1], iters=[20], metric=2, mi_bins=24)
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 20)
    for storage, lt, wt in (("fp64", 1e-5, 1e-4), ("fp32", 1e-6, 1e-5)):
        rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 20, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    assert tr[-1]["loss_raw"] > tr[0]["loss_raw"]  # MI increases


def test_mi_slab_group_bit_identical(P, ctx):
    """MI over z-slabs: the slabs' fixed-point histograms are summed exactly,
    so any split gives the single-domain trajectory bit for bit."""
    F, M, _ = O.synth_pair((20, 24, 28), 24, num_blobs=8, warp_max=2.5)
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[8], metric=2, mi_bins=20)
    w1, (t1,), _ = run_engine(P, ctx, F, M, cfg, 8)
    for ns in (2, 3):
        w, t, _ = run_slabs(P, ctx, F, M, cfg, 8, ns)
        assert same_trace(t, t1) and np.array_equal(w, w1[0]), ns


@pytest.mark.parametrize("extra", [{"metric": 1}, {"metric": 1, "optimizer": 3},
                                   {"metric": 2, "mi_bins": 24}, {"lm.tile_size": 2}])
def test_register_pyramid_other_losses_and_steps(P, ctx, extra):
    """The whole pyramid (levels, warp inheritance, lambda carry) with MSE,
    Demons, MI and tiled LM against the fp32-storage oracle."""
    F, M, _ = O.synth_pair((32, 40, 48), 3, num_blobs=10, warp_max=3.0)
    kw = dict(nlevels=2, factors=[2, 1], iters=[12, 8], **extra)
    res = P.register(F, M, P.reg_config(**kw), ctx=ctx)
    with O.fp32_storage():
        rc, w_s, tr_s, _ = O.register(F, M, O.default_config(**kw))
    assert rc == 0 and len(res.loss_trace) == len(tr_s) == 20
    compare_runs(res.loss_trace, tr_s, res.final_warp, w_s, 1e-6, 1e-5)


def test_bench_json_contract():
    """bench.py's one-line JSON keeps the driver's contract (small config)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--size", "64", "--pairs-per-gpu", "2", "--no-cpu-baseline", "--no-extra",
                          "--e2e-iters", "2"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1 and rf["peak"] > 0 and rf["unit"] == "GB/s"
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0 and e2e["value"] > 0
    # K2, K3, K4, K1a, K1b, plane sums, K5 per attempt and pair group (2 groups of 1 pair
    # here), plus the iteration-target kernel of the one iterate() call
    assert line["gpu_launches"] == 7 * 2 * 3 + 1


def test_bench_two_ranks_under_torchrun():
    """The driver's N > 1 launch (torchrun, one process per rank) end to end:
    one JSON line from rank 0 with the aggregate over ranks.  This box has
    one GPU, so the two ranks share it over a gloo group
    (WLM_BENCH_BACKEND=gloo); the value is not a scaling number."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WLM_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533",
                          os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--size", "64", "--pairs-per-gpu", "2", "--no-cpu-baseline", "--no-extra",
                          "--e2e-iters", "2"], capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 4 and line["value"] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] == 7 * 2 * 3 + 1


def _fuzz_case(i):
    """Seeded random (shape, config) for the engine-vs-oracle sweep."""
    rng = np.random.default_rng(1000 + i)
    shape = tuple(int(v) for v in rng.integers(6, 26, size=3))
    metric = int(rng.choice([0, 0, 1, 2])) if min(shape) > 4 else int(rng.choice([1, 2]))
    optimizer = int(rng.choice([0, 0, 0, 1, 2, 3] if metric == 1 else [0, 0, 0, 1, 2]))
    kw = dict(nlevels=1, factors=[1], iters=[8], metric=metric, optimizer=optimizer,
              sigma_update=float(rng.choice([0.0, 0.7, 1.0, 1.0, 1.3, 1.5, 2.0])),
              sigma_warp=float(rng.choice([0.0, 0.5, 0.5, 0.8, 1.6])))
    if optimizer == 0:
        kw["lm.rejection"] = int(rng.integers(0, 2))
        kw["lm.tau"] = float(rng.choice([0.0, 0.2, 1.0]))
        kw["lm.lambda0"] = float(rng.choice([1e-4, 0.006, 0.5]))
        kw["lm.tile_size"] = int(rng.choice([1, 1, 2, 3]))
    if metric == 2:
        kw["mi_bins"] = int(rng.choice([8, 16, 32]))
    warp_max = float(rng.uniform(0.5, min(shape) / 4 - 0.1))
    return shape, kw, warp_max, int(rng.integers(0, 1 << 30))


@pytest.mark.parametrize("case", range(24))
def test_random_configs_match_storage_oracle(P, ctx, case):
    """Seeded sweep over shapes (ragged, thin), losses, optimizers, rejection,
    damping, tile sizes and smoothing sigmas: the engine against the
    fp32-storage oracle at the storage bar (loss 1e-6, decisions and lambda
    identical, warp 1e-5)."""
    shape, kw, warp_max, seed = _fuzz_case(case)
    for attempt in range(6):  # thin volumes: halve warp_max until a diffeomorphic draw
        try:
            F, M, _ = O.synth_pair(shape, seed, num_blobs=6, warp_max=warp_max / 2 ** attempt)
            break
        except ValueError:
            continue
    else:
        raise AssertionError("synth: no positive-Jacobian draw")
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 8)
    rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 8, "fp32")
    assert rc == 0
    compare_runs(tr, tr_o, aos(warp[0]), u_o, 1e-6, 1e-5)


def _fuzz_generic_case(i):
    """Seeded random configs for the generic device paths (LNCC radius != 2,
    sigma > 2) and the low-memory layout, with the optimizers, rejection and
    tiled LM."""
    rng = np.random.default_rng(5000 + i)
    radius = int(rng.choice([1, 2, 3]))
    shape = tuple(int(v) for v in rng.integers(2 * radius + 3, 24, size=3))
    optimizer = int(rng.choice([0, 0, 1, 2]))
    kw = dict(nlevels=1, factors=[1], iters=[8], optimizer=optimizer, lncc_radius=radius,
              sigma_update=float(rng.choice([1.0, 2.4, 3.0])), sigma_warp=float(rng.choice([0.5, 0.8, 2.2])),
              low_memory=int(rng.integers(0, 2)))
    if optimizer == 0:
        kw["lm.rejection"] = int(rng.integers(0, 2))
        kw["lm.tau"] = float(rng.choice([0.05, 0.3]))
        kw["lm.tile_size"] = int(rng.choice([1, 1, 2]))
    return shape, kw, float(rng.uniform(0.5, min(shape) / 4 - 0.1)), int(rng.integers(0, 1 << 30))


@pytest.mark.parametrize("case", range(12))
def test_random_generic_configs_match_storage_oracle(P, ctx, case):
    """Seeded sweep over the generic paths and the low-memory layout against
    the fp32-storage oracle at the storage bar (loss 1e-6, decisions and
    lambda identical, warp 1e-5)."""
    shape, kw, warp_max, seed = _fuzz_generic_case(case)
    for attempt in range(6):
        try:
            F, M, _ = O.synth_pair(shape, seed, num_blobs=6, warp_max=warp_max / 2 ** attempt)
            break
        except ValueError:
            continue
    else:
        raise AssertionError("synth: no positive-Jacobian draw")
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 8)
    okw = {k: v for k, v in kw.items() if k != "low_memory"}
    rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**okw), 8, "fp32")
    assert rc == 0
    compare_runs(tr, tr_o, aos(warp[0]), u_o, 1e-6, 1e-5)


@pytest.mark.parametrize("su,sw", [(3.0, 0.5), (1.0, 2.5), (2.6, 3.1)])
def test_large_sigma_engine_vs_oracle(P, ctx, su, sw):
    """sigma_update / sigma_warp > 2 (radius > 6: generic.cu's Gaussian passes,
    the reference's gaussian_smooth takes any sigma > 0, field.cpp:205-213)
    against the fp32-storage oracle (loss 1e-6, identical decisions and
    lambda, warp 1e-5) and the fp64 oracle (loss 1e-5).  Slab groups refuse
    these radii (single-domain paths)."""
    F, M, _ = O.synth_pair((26, 30, 34), 41, num_blobs=8, warp_max=2.5)
    kw = dict(nlevels=1, factors=[1], iters=[15], sigma_update=su, sigma_warp=sw,
              **{"lm.rejection": 1, "lm.tau": 0.3})
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 15)
    for storage, lt, wt in (("fp32", 1e-6, 1e-5), ("fp64", 1e-5, 1e-4)):
        rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 15, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    with pytest.raises(P.WlmError):
        P.SlabGroup((26, 30, 34), 2, cfg=P.reg_config(**kw), ctx=ctx)


@pytest.mark.parametrize("radius", [1, 3, 4])
def test_lncc_any_radius_vs_oracle(P, ctx, radius):
    """lncc_radius >= 1: the residual mirror and a
    rejection-on LM run (generic.cu's window passes for radius != 2)
    against the oracle."""
    F, M, _ = O.synth_pair((24, 28, 22), 50 + radius, num_blobs=8, warp_max=2.0)
    F64, M64 = F.astype(np.float64), M.astype(np.float64)
    u = smooth_field(F.shape, 9, sigma=1.5, amp=1.5).astype(np.float32).astype(np.float64)
    rep = P.residual_lncc(F64, M64, u, radius=radius, ctx=ctx)
    r_o, g_o, lncc_o = O.residual_lncc(F64, M64, u, radius=radius)
    assert abs(rep.r - r_o) <= 1e-9 * abs(r_o) and rel(rep.g, g_o) < 1e-6
    kw = dict(nlevels=1, factors=[1], iters=[12], lncc_radius=radius, **{"lm.rejection": 1, "lm.tau": 0.3})
    warp, (tr,), _ = run_engine(P, ctx, F, M, P.reg_config(**kw), 12)
    for storage, lt, wt in (("fp32", 1e-6, 1e-5), ("fp64", 1e-5, 1e-4)):
        rc, u_o, _, tr_o = oracle_level(F, M, O.default_config(**kw), 12, storage)
        assert rc == 0
        compare_runs(tr, tr_o, aos(warp[0]), u_o, lt, wt)
    with pytest.raises(P.InvalidArgument):
        P.Engine(F.shape, 1, P.reg_config(lncc_radius=0), ctx=ctx)


@pytest.mark.parametrize("case", range(12))
def test_random_configs_slab_invariance(P, ctx, case):
    """The same seeded sweep through z-slab groups: any feasible slab count
    reproduces the single-domain engine bit for bit."""
    shape, kw, warp_max, seed = _fuzz_case(100 + case)
    shape = (max(shape[0], 24),) + shape[1:]  # room for >= 2 slabs of the widest halo + tile
    for attempt in range(6):
        try:
            F, M, _ = O.synth_pair(shape, seed, num_blobs=6, warp_max=warp_max / 2 ** attempt)
            break
        except ValueError:
            continue
    else:
        raise AssertionError("synth: no positive-Jacobian draw")
    cfg = P.reg_config(**kw)
    w1, (t1,), _ = run_engine(P, ctx, F, M, cfg, 8)
    tested = 0
    for ns in (2, 3, 4):
        try:
            w, t, _ = run_slabs(P, ctx, F, M, cfg, 8, ns)
        except P.InvalidArgument:
            continue  # slabs thinner than the halo / tile: refused by design
        assert same_trace(t, t1), (ns, kw)
        assert np.array_equal(w, w1[0]), (ns, kw)
        tested += 1
    assert tested > 0


@pytest.mark.parametrize("case", range(10))
def test_random_pyramids_match_storage_oracle(P, ctx, case):
    """Seeded random pyramids through wlm_register (levels, warp inheritance,
    lambda carry, every loss / optimizer of the sweep) against the
    fp32-storage oracle's register, whole trace at the storage bar."""
    shape, kw, warp_max, seed = _fuzz_case(200 + case)
    rng = np.random.default_rng(300 + case)
    shape = tuple(max(s, 12) for s in shape)
    sched = [[2, 1], [3, 1], [4, 2, 1]][int(rng.integers(0, 3))]
    kw = dict(kw, nlevels=len(sched), factors=sched, iters=[int(rng.integers(3, 9)) for _ in sched])
    if kw["metric"] == 0 and any(-(-s // sched[0]) <= 4 for s in shape):
        kw["metric"] = 1  # the coarsest level must fit an LNCC window
        if kw["optimizer"] == 3:
            kw["optimizer"] = 0
    for attempt in range(6):
        try:
            F, M, _ = O.synth_pair(shape, seed, num_blobs=6, warp_max=warp_max / 2 ** attempt)
            break
        except ValueError:
            continue
    else:
        raise AssertionError("synth: no positive-Jacobian draw")
    res = P.register(F, M, P.reg_config(**kw), ctx=ctx)
    with O.fp32_storage():
        rc, w_s, tr_s, _ = O.register(F, M, O.default_config(**kw))
    assert rc == 0 and len(res.loss_trace) == len(tr_s) == sum(kw["iters"])
    for a, b in zip(res.loss_trace, tr_s):
        assert (a.level, a.iter) == (b.level, b.iter)
    compare_runs(res.loss_trace, tr_s, res.final_warp, w_s, 1e-6, 1e-5)


@pytest.mark.parametrize("case", range(12))
def test_random_field_ops_match_oracle(P, ctx, case):
    """Seeded random shapes, fields and sigmas through the host-buffer
    mirrors of field.hpp and the SPEC residuals, against the oracle."""
    rng = np.random.default_rng(500 + case)
    shape = tuple(int(v) for v in rng.integers(5, 20, size=3))
    u = smooth_field(shape, 600 + case, sigma=1.5, amp=float(rng.uniform(0.3, 3.0)))
    v = smooth_field(shape, 700 + case, sigma=1.0, amp=1.0)
    eps = float(rng.uniform(0.05, 0.4))
    # the field mirrors: the reference's bits (fp64 data, its operation order)
    assert same_bits(P.compose_warp(u, v, eps, ctx=ctx), O.compose_warp(u, v, eps))
    sig = float(rng.choice([0.3, 0.5, 1.0, 1.7, 2.5, 3.4]))
    assert same_bits(P.gaussian_smooth(u, sig, ctx=ctx), O.gaussian_smooth(u, sig))
    assert P.max_abs_component(u, ctx=ctx) == O.max_abs_component(u)
    assert P.jacobian_det_min(u, ctx=ctx) == O.jacobian_det_min(u)
    u = u.astype(np.float32).astype(np.float64)  # the residuals take fp32 fields (device storage)
    F = O.gaussian_smooth(rng.normal(size=shape), 1.0).astype(np.float32).astype(np.float64)
    M = O.gaussian_smooth(rng.normal(size=shape), 1.0).astype(np.float32).astype(np.float64)
    r_o, g_o = O.residual_mse(F, M, u)
    rep = P.residual_mse(F, M, u, ctx=ctx)
    assert abs(rep.r - r_o) <= 1e-5 * abs(r_o) and rel(rep.g, g_o) < 1e-4
    r_o, g_o = O.residual_mi(F, M, u, bins=16, sigma=1.0)[:2]
    rep = P.residual_mi(F, M, u, bins=16, sigma=1.0, ctx=ctx)
    assert abs(rep.r - r_o) <= 1e-5 * abs(r_o) and rel(rep.g, g_o) < 1e-4
    if min(shape) > 4:
        r_o, g_o, _ = O.residual_lncc(F, M, u)
        rep = P.residual_lncc(F, M, u, ctx=ctx)
        assert abs(rep.r - r_o) <= 1e-5 * abs(r_o) and rel(rep.g, g_o) < 1e-4


@pytest.mark.parametrize("groups", [1, 2])
def test_nonfinite_pair_does_not_disturb_the_batch(P, ctx, groups):
    """A pair whose moving image holds a NaN aborts alone (its
    state reports the non-finite loss) while the other pairs of the batch run
    to the end bit-identically to a batch without it."""
    shape = (20, 24, 28)
    Fs, Ms = zip(*[O.synth_pair(shape, 800 + s, num_blobs=6, warp_max=2.0)[:2] for s in range(3)])
    F, M = np.stack(Fs), np.stack(Ms).copy()
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[10])
    ref, ref_tr = {}, {}
    for p in (0, 2):
        w, (tr,), _ = run_engine(P, ctx, F[p], M[p], cfg, 10)
        ref[p], ref_tr[p] = w[0], tr
    M[1, 5, 6, 7] = np.nan
    eng = P.Engine(shape, pairs=3, cfg=cfg, ctx=ctx)
    eng.set_pair_groups(groups)
    eng.load(F, M)
    eng.set_warp(None)
    eng.begin_level(0)
    eng.iterate(10)
    warps = eng.get_warp()
    for p in (0, 2):
        assert np.array_equal(warps[p], ref[p]) and same_trace(eng.trace(p), ref_tr[p])
    with pytest.raises(P.NonFiniteLoss):
        eng.state(1)
    assert len(eng.trace(1)) < 10
    eng.close()


def test_batch_pipeline_matches_sequential_runs(P, ctx):
    """BatchPipeline (two engines alternating, copies overlapped) returns
    exactly the warps of running each batch alone."""
    shape = (20, 24, 28)
    batches = []
    for b in range(3):
        pr = [O.synth_pair(shape, 900 + 2 * b + i, num_blobs=6, warp_max=2.0)[:2] for i in range(2)]
        batches.append((np.stack([p[0] for p in pr]), np.stack([p[1] for p in pr])))
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[9])
    pipe = P.BatchPipeline(shape, 2, cfg, iters=9)
    got = list(pipe.run(batches))
    pipe.close()
    assert len(got) == 3
    for (F, M), w in zip(batches, got):
        ref, _, _ = run_engine(P, ctx, F, M, cfg, 9, pairs=2)
        assert np.array_equal(w, ref)


@pytest.mark.parametrize("opt", ["lm", "adam"])
def test_reused_engine_and_slab_group_reset(P, ctx, opt):
    """A second registration on a reused engine or slab group equals a fresh
    one after reset(); without it lambda carries over (SPEC.md:389 carry).
    With Adam, reset() also zeroes the moments (k_adam's bias correction
    restarts at t = 1; stale m, v would be amplified)."""
    shape = (20, 24, 28)
    A = O.synth_pair(shape, 950, num_blobs=6, warp_max=2.0)[:2]
    Bp = O.synth_pair(shape, 951, num_blobs=6, warp_max=2.0)[:2]
    extra = {"optimizer": P.OPT_ADAM} if opt == "adam" else {}
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[8], **extra)
    fresh, (tr_f,), _ = run_engine(P, ctx, Bp[0], Bp[1], cfg, 8)
    for make in (lambda: P.Engine(shape, 1, cfg, ctx=ctx), lambda: P.SlabGroup(shape, 2, cfg=cfg, ctx=ctx)):
        g = make()
        for F, M in (A, Bp):
            g.load(F[None] if isinstance(g, P.Engine) else F, M[None] if isinstance(g, P.Engine) else M)
            g.set_warp(None)
            g.reset()
            g.begin_level(0)
            g.iterate(8)
        w = g.get_warp()
        w = w[0] if isinstance(g, P.Engine) else w
        assert np.array_equal(w, fresh[0])
        g.close()


# ------------------------------------------------- BASELINE's full size ----
@pytest.fixture(scope="module")
def full_pairs():
    """Config 4's volume size (192^3, BASELINE.json configs[3]), seeds 1000
    and 1001 as in bench.py's reference arm."""
    return [O.synth_pair((192, 192, 192), 1000 + s, num_blobs=12, warp_max=6.0)[:2] for s in range(2)]


def test_config4_full_size_vs_oracle(P, ctx, full_pairs):
    """The parity bar at the bench's own size: 4 LM iterations of one 192^3
    pair against the fp32-storage oracle (the tight bar: loss 1e-6, warp
    rel-L2 1e-5; measured 1e-15 / 1.9e-10) and the pure fp64 oracle (loss
    1e-5, same decisions and lambda).  Against fp64 the warp bar is the
    storage floor itself: at 192^3 with 6-voxel displacements, fp32 storage
    of u moves a few hundred sample points across a trilinear knot, where
    grad M jumps, so the fp32-storage oracle is already 4.3e-4 (rel-L2) from
    the fp64 one after 4 iterations (1 iteration: 4.4e-8); the device must
    sit on that floor, not beyond it."""
    F, M = full_pairs[0]
    it = 4
    cfg_p = P.reg_config(nlevels=1, factors=[1], iters=[it])
    cfg_o = O.default_config(nlevels=1, factors=[1], iters=[it])
    warp, (tr,), _ = run_engine(P, ctx, F, M, cfg_p, it)
    w = aos(warp[0])
    rc, u32, _, tr32 = oracle_level(F, M, cfg_o, it, "fp32")
    assert rc == 0
    compare_runs(tr, tr32, w, u32, 1e-6, 1e-5)
    rc, u64, _, tr64 = oracle_level(F, M, cfg_o, it, "fp64")
    assert rc == 0
    compare_runs(tr, tr64, w, u64, 1e-5, None)
    floor = rel(u32, u64)
    assert rel(w, u64) <= floor * (1 + 1e-3) + 1e-6, (rel(w, u64), floor)


def test_config4_full_size_batch_and_slab_invariance(P, ctx, full_pairs):
    """Size-independent properties at 192^3: a pair's result does not depend
    on its batch (bit-identical to the single-pair run) nor on a 4-slab z
    split (config 5's decomposition), over 10 iterations."""
    Fs = np.stack([p[0] for p in full_pairs])
    Ms = np.stack([p[1] for p in full_pairs])
    it = 10
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[it])
    wb, trb, _ = run_engine(P, ctx, Fs, Ms, cfg, it, pairs=2)
    for s in range(2):
        w1, (t1,), _ = run_engine(P, ctx, Fs[s], Ms[s], cfg, it)
        assert np.array_equal(w1[0], wb[s]) and same_trace(t1, trb[s]), s
    w, t, _ = run_slabs(P, ctx, Fs[0], Ms[0], cfg, it, 4)
    assert same_trace(t, trb[0]) and np.array_equal(w, wb[0])


@pytest.mark.parametrize("n,nslabs", [(512, 4), (1024, 2)])
def test_config5_large_slab_split_bit_identical(P, ctx, n, nslabs):
    """Config 5's decomposition at the north star's sizes (512^3 and the
    config's own 1024^3): the GPU synth_pair (seed 7, 96 blobs, max
    displacement 16, as bench.py --config 5), one slab against a z-slab
    split over 3 LM iterations: losses, decisions, lambda and the whole warp
    bit-identical, compared on the device (1024^3 peaks near 120 GB)."""
    import ctypes as C

    import torch
    from paper_2603_19371_b200._lib import Dims, SynthSpec
    shape = (n, n, n)
    F = torch.empty(shape, dtype=torch.float32, device="cuda:0")
    M = torch.empty(shape, dtype=torch.float32, device="cuda:0")
    spec = SynthSpec(Dims(n, n, n), 96, 0.0, 16.0, 0.01, 7)
    ctx.check(P.load().wlm_synth_pair(ctx.h, C.byref(spec), F.data_ptr(), M.data_ptr(), None, 1))
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[3])
    out = {}
    for ns in (1, nslabs):
        grp = P.SlabGroup(shape, ns, cfg=cfg, ctx=ctx)
        grp.load(F, M)
        grp.set_warp(None)
        grp.begin_level(0)
        grp.iterate(3)
        w = torch.zeros((3,) + shape, dtype=torch.float32, device="cuda:0")
        grp.get_warp(w)
        out[ns] = (w, grp.trace(), grp.state())
        grp.close()
        del grp
    (w1, t1, s1), (w4, t4, s4) = out[1], out[nslabs]
    assert len(t1) >= 3 and all(math.isfinite(r["r"]) for r in t1)
    assert same_trace(t4, t1) and s4["lam"] == s1["lam"] and s4["r"] == s1["r"]
    assert bool(torch.equal(w1, w4)) and float(w1.abs().max()) > 0.0


@pytest.mark.parametrize("rejection", [0, 1])
def test_low_memory_layout_is_bit_identical(P, ctx, rejection):
    """low_memory = 1 (no fp64 grad M buffer; K2 re-gathers M at x + u with
    K1a's arithmetic) gives the default layout's warps and traces bit for
    bit, through the batch engine and the pyramid driver, and holds 24 B
    per voxel less device memory (the grad M buffer)."""
    shape = (26, 30, 34)
    F, M, _ = O.synth_pair(shape, 61, num_blobs=8, warp_max=2.5)
    kw = dict(nlevels=1, factors=[1], iters=[20], **{"lm.rejection": rejection, "lm.tau": 0.05})
    out = {}
    for lean in (0, 1):
        w, (t,), _ = run_engine(P, ctx, F, M, P.reg_config(low_memory=lean, **kw), 20)
        out[lean] = (w, t)
    assert np.array_equal(out[0][0], out[1][0]) and same_trace(out[0][1], out[1][1])
    if rejection:
        assert sum(r["retries"] for r in out[0][1]) > 0
    kw = dict(nlevels=2, factors=[2, 1], iters=[15, 10])
    res = {lean: P.register(F, M, P.reg_config(low_memory=lean, **kw), ctx=ctx) for lean in (0, 1)}
    assert np.array_equal(res[0].final_warp, res[1].final_warp)
    assert [(a.r, a.lam) for a in res[0].loss_trace] == [(a.r, a.lam) for a in res[1].loss_trace]
    assert res[0].peak_device_bytes - res[1].peak_device_bytes == 24 * int(np.prod(shape))
