"""CPU tests: pin the oracle (test infrastructure) before trusting it.

1. Bit-for-bit against golden vectors produced by the UNMODIFIED reference
   field.cpp (tests/golden/make_golden.py via oracle/_ref).
2. Bit-for-bit against the live reference when oracle/_ref is built.
3. Every SPEC known-answer example and property for the path (SPEC.md lines
   cited per test).
"""
import math

import numpy as np
import pytest

import oracle as O
from conftest import rel, smooth_field


# ---------------------------------------------------------------- golden ----
def test_golden_sample_trilinear_grad(golden):
    vol, pts = golden["sample_vol"], golden["sample_pts"]
    for q, v, g in zip(pts, golden["sample_val"], golden["sample_grad"]):
        val, gr = O.sample_trilinear_grad(vol, q)
        if math.isnan(v):
            assert math.isnan(val)
        else:
            assert val == v
            assert np.array_equal(gr, g)


@pytest.mark.parametrize("name", ["c6", "c876"])
def test_golden_compose(golden, name):
    out = O.compose_warp(golden[f"{name}_u"], golden[f"{name}_v"], float(golden[f"{name}_eps"]))
    assert np.array_equal(out, golden[f"{name}_out"])


@pytest.mark.parametrize("key", ["1p0", "0p5", "2p3"])
def test_golden_smooth(golden, key):
    sig = float(key.replace("p", "."))
    assert np.array_equal(O.gaussian_smooth(golden[f"sm{key}_field_in"], sig), golden[f"sm{key}_field_out"])
    assert np.array_equal(O.gaussian_smooth(golden[f"sm{key}_vol_in"], sig), golden[f"sm{key}_vol_out"])


def test_golden_jac_max_norm(golden):
    assert O.jacobian_det_min(golden["jac_u"]) == float(golden["jac_out"])
    assert O.jacobian_det_min(golden["jac2_u"]) == float(golden["jac2_out"])
    assert O.max_abs_component(golden["jac_u"]) == float(golden["max_out"])
    assert O.normalize_step(golden["jac_u"]) == float(golden["norm_out"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference here)")
def test_oracle_matches_live_reference():
    L = O.ref_lib()
    rng = np.random.default_rng(7)
    u = rng.normal(size=(9, 10, 11, 3))
    v = rng.normal(size=(9, 10, 11, 3))
    o = np.empty_like(u)
    L.ref_compose_warp(O._p(u), 11, 10, 9, O._p(v), 11, 10, 9, 0.37, O._p(o))
    assert np.array_equal(O.compose_warp(u, v, 0.37), o)
    w = u.copy()
    L.ref_gaussian_smooth(O._p(w), 11, 10, 9, 3, 1.0)
    assert np.array_equal(O.gaussian_smooth(u, 1.0), w)
    M = rng.normal(size=(9, 10, 11))
    Mw, gM = O.warp_volume(M, u)
    Mr, gr = np.empty_like(M), np.empty_like(u)
    L.ref_warp_volume(O._p(M), O._p(u), 11, 10, 9, O._p(Mr), O._p(gr))
    assert np.array_equal(Mw, Mr) and np.array_equal(gM, gr)
    # the "reference" build routes field primitives through field.cpp itself
    F = rng.uniform(size=(12, 12, 12))
    Mv = rng.uniform(size=(12, 12, 12))
    uu = smooth_field((12, 12, 12), 3, amp=1.2)
    a = O.residual_lncc(F, Mv, uu)[0]
    b = O.residual_lncc(F, Mv, uu, kind="reference")[0]
    assert a == b


# ------------------------------------------------------------- SPEC KATs ----
def test_sample_kats():
    # SPEC.md:53-55
    assert O.sample_trilinear_grad(np.full((9, 9, 9), 5.0), (0.3, 7.9, 2.1))[0] == 5.0
    v = np.zeros((4, 4, 4)); v[0, 0, 1] = 1.0
    assert O.sample_trilinear_grad(v, (0.25, 0, 0))[0] == 0.25
    ramp = np.broadcast_to(np.arange(4.0)[None, None, :], (4, 4, 4)).copy()
    assert O.sample_trilinear_grad(ramp, (5.0, 0, 0))[0] == 3.0
    # SPEC.md:87 exact at integer points
    rng = np.random.default_rng(0)
    vol = rng.normal(size=(5, 5, 5))
    for z, y, x in [(0, 0, 0), (4, 4, 4), (2, 3, 1)]:
        assert abs(O.sample_trilinear_grad(vol, (x, y, z))[0] - vol[z, y, x]) < 1e-12


def test_compose_kats():
    rng = np.random.default_rng(1)
    v = rng.normal(size=(6, 6, 6, 3))
    assert np.array_equal(O.compose_warp(np.zeros_like(v), v, 0.1), 0.1 * v)
    c = np.broadcast_to(np.array([0.3, -1.2, 2.0]), (6, 6, 6, 3)).copy()
    assert np.allclose(O.compose_warp(c, np.zeros_like(c), 0.5), c, atol=0)


def test_normalize_and_jacobian_kats():
    v = np.zeros((4, 4, 4, 3)); v[1, 2, 3, 0] = -2.0
    assert O.normalize_step(v) == pytest.approx(0.2)
    assert math.isnan(O.normalize_step(v, target=0.6))  # field.cpp:151-153
    u0 = np.zeros((5, 5, 5, 3))
    assert O.jacobian_det_min(u0) == 1.0
    assert O.jacobian_det_min(u0 + np.array([1.0, 2.0, -3.0])) == 1.0
    ramp = u0.copy(); ramp[..., 0] = 0.1 * np.arange(5)[None, None, :]
    assert O.jacobian_det_min(ramp) == pytest.approx(1.1, abs=1e-12)


def test_lncc_kats():
    F, M, _ = O.synth_pair((16, 16, 16), 5, warp_max=0.0, noise_sigma=0.05)
    F = F.astype(np.float64)
    r, g, lncc = O.residual_lncc(F, 2 * F + 3, np.zeros(F.shape + (3,)))
    assert abs(lncc - 1.0) < 1e-9 and abs(r) < 1e-9
    r, g, lncc = O.residual_lncc(np.full((10, 10, 10), 0.7), F[:10, :10, :10], np.zeros((10, 10, 10, 3)))
    assert lncc == 0.0 and r == 1.0 and not g.any()
    assert math.isnan(O.residual_lncc(F[:4], F[:4], np.zeros(F[:4].shape + (3,)))[0])


def _fd_check(fn, F, M, u, n=30, h=1e-4, seed=0):
    r0, g = fn(F, M, u)[:2]
    rng = np.random.default_rng(seed)
    idx = [tuple(rng.integers(0, s) for s in u.shape) for _ in range(n)]
    errs = []
    for i in idx:
        up = u.copy(); up[i] += h
        um = u.copy(); um[i] -= h
        fd = (fn(F, M, up)[0] - fn(F, M, um)[0]) / (2 * h)
        errs.append(abs(fd - g[i]) / max(abs(fd), abs(g[i]), 1e-30))
    return np.array(errs), g


def test_lncc_gradient_finite_differences():
    # SPEC.md:144 / :156: random smooth 12^3 pair, 30 components, rel < 1e-3
    rng = np.random.default_rng(3)
    F = O.gaussian_smooth(rng.uniform(size=(12, 12, 12)), 1.0)
    M = O.gaussian_smooth(rng.uniform(size=(12, 12, 12)), 1.0)
    u = smooth_field((12, 12, 12), 4, amp=0.7) + 0.123  # off the knots
    errs, g = _fd_check(lambda a, b, c: O.residual_lncc(a, b, c), F, M, u)
    big = np.abs(g).max()
    # components whose gradient is ~0 are compared absolutely
    assert np.all((errs < 1e-3)), errs


def test_mse_gradient_finite_differences():
    rng = np.random.default_rng(8)
    F = O.gaussian_smooth(rng.uniform(size=(8, 8, 8)), 1.0)
    M = O.gaussian_smooth(rng.uniform(size=(8, 8, 8)), 1.0)
    u = smooth_field((8, 8, 8), 9, amp=0.6) + 0.31
    errs, _ = _fd_check(O.residual_mse, F, M, u)
    assert np.all(errs < 1e-4), errs


def test_mse_kats():
    """aligned pair -> 0; constant offset -> 1; at u = 0
    r equals the plain mean-squared difference (independent one-liner)."""
    rng = np.random.default_rng(4)
    F = rng.uniform(size=(6, 7, 8))
    z = np.zeros(F.shape + (3,))
    r, g = O.residual_mse(F, F, z)
    assert r == 0.0 and not g.any()
    r, _ = O.residual_mse(np.zeros_like(F), np.ones_like(F), z)
    assert r == 1.0
    M = rng.uniform(size=F.shape)
    r, _ = O.residual_mse(F, M, z)
    assert abs(r - np.mean((F - M) ** 2)) <= 1e-12


def test_mse_lm_iterate_decreases_loss():
    """lm_run_level with MetricConfig.kind = mse: r = loss_raw."""
    F, M, _ = O.synth_pair((16, 16, 16), 2, num_blobs=6, warp_max=1.5)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[15], metric=1)
    rc, u, st, tr = O.lm_run_level(F, M, np.zeros((16, 16, 16, 3)), cfg, 15)
    assert rc == 0 and len(tr) == 15
    assert all(t.r == t.loss_raw for t in tr)
    r0, _ = O.residual_mse(F, M, np.zeros((16, 16, 16, 3)))
    assert tr[-1].r < 0.8 * r0


def test_mi_kats_and_bounds():
    """SPEC.md:150-153, :157-159.  Identical images with B levels on the bin
    centres reach MI ~ log2 B when the Parzen kernel is narrow (sigma = 0.25
    bin; at the default sigma = 1 the kernel blurs adjacent levels, DESIGN.md
    A16); independent noise -> MI < 0.1 bits at 32^3; 0 <= MI <= log2 B."""
    rng = np.random.default_rng(0)
    B = 32
    F = np.repeat(np.arange(B, dtype=float), 32 ** 3 // B).reshape(32, 32, 32)
    rng.shuffle(F.reshape(-1))
    z = np.zeros(F.shape + (3,))
    r, g, mi = O.residual_mi(F, F, z, bins=B, sigma=0.25)
    assert r < 0.2 and abs(r - (np.log2(B) - mi)) < 1e-12
    r, g, mi = O.residual_mi(rng.uniform(size=(32, 32, 32)), rng.uniform(size=(32, 32, 32)), z)
    assert mi < 0.1
    for seed in range(20):
        q = np.random.default_rng(100 + seed)
        F = q.uniform(size=(6, 6, 6)) ** q.uniform(0.5, 3)
        M = q.normal(size=(6, 6, 6))
        r, _, mi = O.residual_mi(F, M, np.zeros((6, 6, 6, 3)), bins=int(q.integers(2, 40)))
        assert -1e-12 <= mi and r >= -1e-12


def test_mi_gradient_finite_differences():
    rng = np.random.default_rng(6)
    F = O.gaussian_smooth(rng.uniform(size=(10, 10, 10)), 1.0)
    M = O.gaussian_smooth(rng.uniform(size=(10, 10, 10)), 1.0)
    u = smooth_field((10, 10, 10), 3, amp=0.7) + 0.137
    errs, _ = _fd_check(lambda a, b, c: O.residual_mi(a, b, c, bins=16)[:2], F, M, u)
    assert np.all(errs < 1e-3), errs


def _dense_tiled(r, g, lam, k):
    """Independent dense per-tile assemble-and-solve."""
    out = np.empty_like(g)
    nz, ny, nx, _ = g.shape
    for z0 in range(0, nz, k):
        for y0 in range(0, ny, k):
            for x0 in range(0, nx, k):
                blk = g[z0:z0 + k, y0:y0 + k, x0:x0 + k].reshape(-1, 3)
                H = blk.T @ blk + lam * np.eye(3)
                sol = np.linalg.solve(H, -r * blk.T).T
                out[z0:z0 + k, y0:y0 + k, x0:x0 + k] = sol.reshape(g[z0:z0 + k, y0:y0 + k, x0:x0 + k].shape)
    return out


def test_tiled_lm_kats():
    """k = 1 == pointwise to 1e-12; g = 0 -> 0; random
    6^3 and 7^3 (partial tiles), k = 3 (and 2, 4) == dense per-tile solve."""
    rng = np.random.default_rng(21)
    g = rng.normal(size=(5, 6, 7, 3))
    assert np.abs(O.lm_step_tiled(0.7, g, 0.3, 1) - O.lm_step_pointwise(0.7, g, 0.3)).max() < 1e-12
    assert not O.lm_step_tiled(0.7, np.zeros_like(g), 0.3, 3).any()
    for shape, k in (((6, 6, 6), 3), ((7, 7, 7), 3), ((7, 5, 9), 2), ((8, 7, 6), 4)):
        g = rng.normal(size=shape + (3,)) * rng.uniform(0.01, 2.0)
        lam = rng.uniform(0.01, 3.0)
        ref = _dense_tiled(0.4, g, lam, k)
        assert np.abs(O.lm_step_tiled(0.4, g, lam, k) - ref).max() < 1e-10


def test_tiled_lm_iterate():
    F, M, _ = O.synth_pair((16, 16, 16), 5, num_blobs=6, warp_max=1.5)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[10], **{"lm.tile_size": 3})
    rc, u, st, tr = O.lm_run_level(F, M, np.zeros((16, 16, 16, 3)), cfg, 10)
    assert rc == 0 and len(tr) == 10 and tr[-1].r < tr[0].r


def test_demons_kats_and_lm_equivalence():
    """r_x = 0 -> 0; n = (2,0,0), r = 1, alpha = 1
    -> (0.4, 0, 0); equals per-voxel LM with r := r_x, lambda := alpha^2 r_x^2
    (g := -n, the gradient of r_x = f - m(x+u)) to 1e-12."""
    assert not O.demons_step_mse(np.zeros((2, 2, 2)), np.ones((2, 2, 2, 3)), 1.0).any()
    out = O.demons_step_mse(np.ones((1, 1, 1)), np.array([[[[2.0, 0.0, 0.0]]]]), 1.0)
    assert np.allclose(out[0, 0, 0], [0.4, 0.0, 0.0], rtol=0, atol=1e-15)
    # zero denominator (n = 0 and r = 0) -> 0, not NaN
    assert not O.demons_step_mse(np.zeros((1, 1, 1)), np.zeros((1, 1, 1, 3)), 1.0).any()
    rng = np.random.default_rng(17)
    F = O.gaussian_smooth(rng.uniform(size=(8, 9, 10)), 1.0)
    M = O.gaussian_smooth(rng.uniform(size=(8, 9, 10)), 1.0)
    u = smooth_field((8, 9, 10), 5, amp=0.8) + 0.2
    Mw, gM = O.warp_volume(M, u)
    rx = F - Mw
    for alpha in (0.5, 1.0, 2.0):
        d = O.demons_step_mse(rx, gM, alpha)
        lm = np.empty_like(d)
        for i in np.ndindex(rx.shape):
            lm[i] = O.lm_step_pointwise(rx[i], -gM[i].reshape(1, 1, 1, 3), alpha ** 2 * rx[i] ** 2)[0, 0, 0]
        assert np.abs(d - lm).max() < 1e-12


def test_demons_registration_decreases_mse():
    F, M, _ = O.synth_pair((16, 16, 16), 3, num_blobs=6, warp_max=1.5)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[15], metric=1, optimizer=3)
    rc, u, st, tr = O.lm_run_level(F, M, np.zeros((16, 16, 16, 3)), cfg, 15)
    assert rc == 0 and len(tr) == 15 and all(t.lam == 0.0 for t in tr)
    r0, _ = O.residual_mse(F, M, np.zeros((16, 16, 16, 3)))
    assert tr[-1].r < 0.8 * r0


def test_lm_step_kats_and_sherman_morrison():
    g = np.zeros((2, 2, 2, 3)); g[0, 0, 0] = (1, 0, 0)
    out = O.lm_step_pointwise(2.0, g, 1.0)
    assert np.array_equal(out[0, 0, 0], [-1.0, 0.0, 0.0])
    assert not out[1:].any()
    rng = np.random.default_rng(11)  # SPEC.md:255, :321, :481 (1e5 triples)
    G = rng.normal(size=(100000, 3)) * rng.uniform(0.01, 10, size=(100000, 1))
    r = rng.uniform(0.1, 2.0, size=100000)
    lam = 10 ** rng.uniform(-3, 1, size=100000)
    closed = -r[:, None] * G / ((G * G).sum(1) + lam)[:, None]
    A = G[:, :, None] * G[:, None, :] + lam[:, None, None] * np.eye(3)
    dense = np.linalg.solve(A, (-r[:, None] * G)[..., None])[..., 0]
    assert np.abs(closed - dense).max() < 1e-10
    for i in range(50):  # the oracle's own explicit solver
        assert np.allclose(O.lm_step_dense3(r[i], G[i], lam[i]), closed[i], atol=1e-10, rtol=0)
    # GD limit
    gg = rng.normal(size=(3, 3, 3, 3))
    big = 1e8 * (gg ** 2).sum(-1).max()
    assert rel(O.lm_step_pointwise(0.7, gg, big), -0.7 * gg / big) < 1e-6


def test_damping_and_rejection_kats():
    c = O.lm_config()
    s = O.update_damping(O.LmState(0.006, 1, 0.5, 0.0), 0.4, c)  # good step
    assert s.lam == pytest.approx(0.00585, abs=1e-15)
    s = O.update_damping(O.LmState(0.006, 1, 0.5, 0.0), 0.6, c)
    assert s.lam == pytest.approx(0.009, abs=1e-15)
    s = O.update_damping(O.LmState(0.9, 1, 0.5, 0.0), 0.6, c)
    assert s.lam == 1.0
    s = O.update_damping(O.LmState(0.006, 0, 0.0, 0.0), 0.1, c)
    assert s.lam == pytest.approx(0.009)  # no history -> bad
    s = O.update_damping(O.LmState(0.006, 1, 0.5, 0.0), 0.5, c)
    assert s.lam == pytest.approx(0.00585)  # tie is good
    assert O.rejection_test(1.05, 0.9, 1.0, 1.0)
    assert not O.rejection_test(0.85, 0.9, 1.0, 1.0)
    assert not O.rejection_test(0.99, 0.9, 1.0, 1.0)


def test_scripted_lambda_trajectories():
    # 10 forced rejections with cap 1.0
    c = O.lm_config(rejection=1)
    losses = [1.0, 0.9] + [5.0] * 11
    lam, dec, st = O.lm_replay(losses, 3, c)
    assert list(dec) == [0, 0] + [1] * 10 + [0]
    l0 = 0.006 * 1.5 * 0.975  # after the two history-building steps
    assert lam[11] == pytest.approx(min(l0 * 1.5 ** 10, 1.0), rel=1e-15)
    lam, dec, st = O.lm_replay(losses, 3, c, O.LmState(0.3, 0, 0.0, 0.0))
    assert lam[11] == 1.0 and lam.max() == 1.0  # the cap binds exactly
    # alternating good/bad -> lambda0 (mu+ mu-)^m (rejection off)
    c2 = O.lm_config()
    st0 = O.LmState(0.006, 1, 10.0, 0.0)
    seq = []
    L = 10.0
    for k in range(20):
        L = L - 1.0 if k % 2 == 0 else L + 0.5
        seq.append(L)
    lam, dec, st = O.lm_replay(seq, 20, c2, st0)
    for m in range(1, 11):
        assert lam[2 * m - 1] == pytest.approx(0.006 * (1.5 * 0.975) ** m, rel=1e-12)
    # rejection never fires on monotonically decreasing losses
    lam, dec, _ = O.lm_replay(np.linspace(1, 0.1, 30), 30, c)
    assert not dec.any()
    # with the cap, lambda never exceeds lambda_max
    lam, dec, _ = O.lm_replay(np.r_[1.0, 0.9, np.full(200, 3.0)], 50, c)
    assert lam.max() <= 1.0


def test_iterate_integration_16():
    # 16^3, 5 iterations, defaults -> non-increasing in >= 4 of 5
    F, M, _ = O.synth_pair((16, 16, 16), 2, num_blobs=6, warp_max=1.5)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[5], log_jacobian=1)
    rc, u, st, tr = O.lm_run_level(F, M, np.zeros((16, 16, 16, 3)), cfg, 5)
    assert rc == 0 and len(tr) == 5
    rs = [t.r for t in tr]
    assert sum(b <= a for a, b in zip(rs, rs[1:])) >= 3
    assert all(t.jac_det_min > 0 for t in tr)
    assert all(abs(t.eps * 1.0) > 0 for t in tr)


def test_pyramid_kats():
    v = np.full((32, 32, 32), 3.25)
    d = O.downsample(v, 2)
    assert d.shape == (16, 16, 16) and np.abs(d - 3.25).max() < 1e-10
    assert O.downsample(np.ones((9, 7, 5)), 4).shape == (3, 2, 2)  # ceil dims
    # 8^3 ramp, factor 2 vs an independent smooth-then-stride loop
    ramp = np.fromfunction(lambda z, y, x: x + 2 * y - z, (8, 8, 8))
    sm = O.gaussian_smooth(ramp, 1.0)
    assert np.abs(O.downsample(ramp, 2) - sm[::2, ::2, ::2]).max() < 1e-10
    u = np.zeros((8, 8, 8, 3))
    assert not O.upsample_warp(u, (16, 16, 16), 2.0).any()
    t = np.zeros((8, 8, 8, 3)); t[..., 0] = 1.0
    up = O.upsample_warp(t, (16, 16, 16), 2.0)
    assert np.allclose(up[..., 0], 2.0) and not up[..., 1:].any()
    cu = smooth_field((8, 8, 8), 5, sigma=2.0)
    fu = O.upsample_warp(cu, (16, 16, 16), 2.0)
    assert np.abs(fu[::2, ::2, ::2] / 2.0 - cu).max() < 1e-6


def test_adam_kats():
    g = np.full(12, 0.3)
    m = np.zeros(12); v = np.zeros(12)
    out = O.adam_step(g, m, v, 1, lr=0.5)
    assert np.allclose(out, -0.5, atol=1e-6)
    m = np.zeros(12); v = np.zeros(12)
    assert not O.adam_step(np.zeros(12), m, v, 1).any()
    # 3 steps vs an independent scalar implementation
    rng = np.random.default_rng(4)
    gs = rng.normal(size=(3, 24))
    m = np.zeros(24); v = np.zeros(24)
    mm = np.zeros(24); vv = np.zeros(24)
    for t in range(1, 4):
        out = O.adam_step(gs[t - 1], m, v, t)
        mm = 0.9 * mm + 0.1 * gs[t - 1]
        vv = 0.999 * vv + 0.001 * gs[t - 1] ** 2
        ref = -0.5 * (mm / (1 - 0.9 ** t)) / (np.sqrt(vv / (1 - 0.999 ** t)) + 1e-8)
        assert np.abs(out - ref).max() < 1e-12


def test_synth_determinism_and_contract():
    a = O.synth_pair((20, 18, 16), 9, warp_max=2.0)
    b = O.synth_pair((20, 18, 16), 9, warp_max=2.0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    F, M, U = O.synth_pair((20, 18, 16), 3, warp_max=0.0, noise_sigma=0.0)
    assert np.array_equal(F, M) and not U.any()
    F, M, U = O.synth_pair((24, 24, 24), 4, warp_max=2.0)
    assert abs(np.abs(U).max() - 2.0) < 1e-6
    assert O.jacobian_det_min(U.astype(np.float64)) > 0


def test_register_recovers_translation():
    # SPEC.md:369 analogue: blob pair translated by 2 voxels, LM defaults
    F, _, _ = O.synth_pair((24, 24, 24), 12, num_blobs=5, warp_max=0.0, noise_sigma=0.0)
    F = F.astype(np.float64)
    sh = np.zeros(F.shape + (3,)); sh[..., 0] = -2.0
    M, _ = O.warp_volume(F, sh)  # M(x) = F(x - 2 e_x)  ->  solution u = +2 e_x
    cfg = O.default_config(nlevels=3, factors=[4, 2, 1], iters=[40, 30, 20])
    rc, warp, trace, jac = O.register(F.astype(np.float32), M.astype(np.float32), cfg)
    assert rc == 0 and len(trace) == 90
    c = (slice(6, 18),) * 3
    assert np.abs(warp[c][..., 0] - 2.0).mean() < 0.5
    assert jac > 0
