"""Python mirror of the reference ``warplm`` API, backed by the sm_100a library.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/warplm/field.hpp and SPEC.md):

  reference                                  here
  field.hpp:96  compose_warp(u, v, eps)      compose_warp(u, v, eps)       DimensionMismatch
  field.hpp:99  max_abs_component(v)         max_abs_component(v)
  field.hpp:104 normalize_step(v, s)         normalize_step(v, StepScale)  InvalidArgument
  field.hpp:108 jacobian_det_min(u)          jacobian_det_min(u)           InvalidArgument
  field.hpp:113 gaussian_smooth(vol|field)   gaussian_smooth(a, sigma)
  field.hpp:116 all_finite                   all_finite(a)
  field.hpp:90  sample_trilinear_grad        warp_volume(M, u) (whole volume)
  field.hpp:93  sample_field                 sample_field(u, p)
  SPEC.md:136   residual_lncc                residual_lncc(F, M, u, cfg)   -> ResidualReport
  SPEC.md:247   lm_step_pointwise            lm_step_pointwise(r, g, lam)
  SPEC.md:265   update_damping               update_damping(state, loss, cfg)
  SPEC.md:274   rejection_test               rejection_test(new, prev, prev2, tau)
  SPEC.md:188   downsample                   downsample(vol, factor)
  SPEC.md:197   upsample_warp                upsample_warp(u, new_shape, scale)
  SPEC.md:310   state_bytes                  state_bytes(optimizer, shape)
  SPEC.md:362   register                     register(F, M, cfg)           -> RegResult

Array conventions (reference Dims3::index, field.hpp:25-30): a Volume3 is a
float64 array of shape (nz, ny, nx); a DispField3 is (nz, ny, nx, 3),
component innermost (field.hpp:50-58).
"""
from __future__ import annotations

import atexit
import ctypes as C
import weakref
from dataclasses import dataclass, field as dfield

import numpy as np

from ._lib import (AdamConfig, Dims, DimensionMismatch, InvalidArgument, LmConfig, LmState,
                   METRIC_LNCC, METRIC_MI, METRIC_MSE, NonFiniteLoss, OPT_ADAM, OPT_DEMONS, OPT_GD, OPT_LM, RegConfig, StepLog, WlmError, check,
                   load)

__all__ = [
    "Context", "StepScale", "ResidualReport", "RegResult", "compose_warp", "max_abs_component",
    "normalize_step", "jacobian_det_min", "gaussian_smooth", "all_finite", "sample_field",
    "sample_trilinear", "sample_trilinear_grad",
    "warp_volume", "residual_lncc", "lm_step_pointwise", "update_damping", "rejection_test",
    "downsample", "upsample_warp", "state_bytes", "register", "reg_config", "lm_config",
    "DimensionMismatch", "InvalidArgument", "NonFiniteLoss", "WlmError", "OPT_LM", "OPT_ADAM",
    "OPT_GD", "OPT_DEMONS", "LmState", "LmConfig", "METRIC_LNCC", "METRIC_MSE", "METRIC_MI", "residual_mse", "residual_mi",
    "demons_step_mse", "lm_step_tiled", "synth_pair", "trace_rows",
]

_D = C.POINTER(C.c_double)


def _p(a):
    return a.ctypes.data_as(_D)


# Live handles, released in dependency order (engines, then contexts) before
# the CUDA runtime tears down at interpreter exit.
_LIVE_ENGINES: "weakref.WeakSet" = weakref.WeakSet()
_LIVE_CONTEXTS: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _release_all():
    for e in list(_LIVE_ENGINES):
        e.close()
    for c in list(_LIVE_CONTEXTS):
        c.close()


class Context:
    """One wlm_ctx: a CUDA stream + scratch on one device."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        st = self.lib.wlm_ctx_create(device, C.byref(h))
        if st != 0:
            raise WlmError(st, f"wlm_ctx_create(device={device}) failed: no usable CUDA device")
        self.h = h
        _LIVE_CONTEXTS.add(self)

    def check(self, status):
        check(status, self.h)

    @property
    def launches(self) -> int:
        return int(self.lib.wlm_ctx_launch_count(self.h))

    @property
    def peak_bytes(self) -> int:
        return int(self.lib.wlm_ctx_peak_bytes(self.h))

    def synchronize(self):
        self.check(self.lib.wlm_ctx_synchronize(self.h))

    def stream(self) -> int:
        return int(self.lib.wlm_ctx_stream(self.h) or 0)

    def close(self):
        if getattr(self, "h", None):
            self.lib.wlm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _ctx(ctx):
    return ctx or default_context()


def _vol(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 3:
        raise InvalidArgument(1, "Volume3 must be a (nz, ny, nx) array")
    return a


def _fld(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 4 or a.shape[3] != 3:
        raise InvalidArgument(1, "DispField3 must be a (nz, ny, nx, 3) array")
    return a


def _dims(shape) -> Dims:
    return Dims(int(shape[2]), int(shape[1]), int(shape[0]))


@dataclass
class StepScale:
    """field.hpp:75-78."""
    target_max_disp: float = 0.4
    floor: float = 1e-12


@dataclass
class ResidualReport:
    """r, g = dr/du, loss_raw (the LNCC value)."""
    r: float
    g: np.ndarray | None
    loss_raw: float


@dataclass
class RegResult:
    """SPEC.md:356-359."""
    final_warp: np.ndarray
    loss_trace: list = dfield(default_factory=list)
    jac_det_min_final: float = float("nan")
    peak_device_bytes: int = 0


def compose_warp(u, v, eps, ctx=None):
    u, v = _fld(u), _fld(v)
    c = _ctx(ctx)
    out = np.empty_like(u)
    c.check(c.lib.wlm_compose_warp(c.h, _p(u), _dims(u.shape), _p(v), _dims(v.shape), float(eps),
                                   _p(out)))
    return out


def max_abs_component(v, ctx=None):
    v = _fld(v)
    c = _ctx(ctx)
    out = C.c_double()
    c.check(c.lib.wlm_max_abs_component(c.h, _p(v), _dims(v.shape), C.byref(out)))
    return out.value


def normalize_step(v, s: StepScale = StepScale(), ctx=None):
    v = _fld(v)
    c = _ctx(ctx)
    out = C.c_double()
    c.check(c.lib.wlm_normalize_step(c.h, _p(v), _dims(v.shape), float(s.target_max_disp),
                                     float(s.floor), C.byref(out)))
    return out.value


def jacobian_det_min(u, ctx=None):
    u = _fld(u)
    c = _ctx(ctx)
    out = C.c_double()
    c.check(c.lib.wlm_jacobian_det_min(c.h, _p(u), _dims(u.shape), C.byref(out)))
    return out.value


def gaussian_smooth(a, sigma, ctx=None):
    c = _ctx(ctx)
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty_like(a)
    if a.ndim == 3:
        c.check(c.lib.wlm_gaussian_smooth_vol(c.h, _p(a), _dims(a.shape), float(sigma), _p(out)))
    else:
        a = _fld(a)
        c.check(c.lib.wlm_gaussian_smooth_field(c.h, _p(a), _dims(a.shape), float(sigma), _p(out)))
    return out


def all_finite(a, ctx=None) -> bool:
    c = _ctx(ctx)
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = C.c_int()
    c.check(c.lib.wlm_all_finite(c.h, _p(a), a.size, C.byref(out)))
    return bool(out.value)


def sample_trilinear_grad(vol, points, ctx=None):
    """sample_trilinear_grad (field.cpp:47-90) at N points (x, y, z): values
    (N,) and analytic gradients (N, 3); NaN value for a non-finite point."""
    vol = _vol(vol)
    pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
    c = _ctx(ctx)
    val = np.empty(pts.shape[0])
    grad = np.empty_like(pts)
    c.check(c.lib.wlm_sample_trilinear_grad_points(c.h, _p(vol), _dims(vol.shape), _p(pts), pts.shape[0],
                                                   _p(val), _p(grad)))
    return val, grad


def sample_trilinear(vol, points, ctx=None):
    """sample_trilinear (field.cpp:43-45) at N points."""
    return sample_trilinear_grad(vol, points, ctx=ctx)[0]


def sample_field(u, points, ctx=None):
    u = _fld(u)
    pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
    c = _ctx(ctx)
    out = np.empty_like(pts)
    c.check(c.lib.wlm_sample_field_points(c.h, _p(u), _dims(u.shape), _p(pts), pts.shape[0], _p(out)))
    return out


def warp_volume(M, u, ctx=None):
    """M(x + u(x)) and the analytic interpolant gradient (field.cpp:47-90)."""
    M, u = _vol(M), _fld(u)
    if u.shape[:3] != M.shape:
        raise DimensionMismatch(2, "warp_volume: dimension mismatch")
    c = _ctx(ctx)
    Mw = np.empty_like(M)
    gM = np.empty(M.shape + (3,))
    c.check(c.lib.wlm_warp_volume(c.h, _p(M), _p(u), _dims(M.shape), _p(Mw), _p(gM)))
    return Mw, gM


def residual_lncc(F, M, u, radius=2, gradient=True, ctx=None) -> ResidualReport:
    F, M, u = _vol(F), _vol(M), _fld(u)
    if F.shape != M.shape or u.shape[:3] != F.shape:
        raise DimensionMismatch(2, "residual_lncc: dimension mismatch")
    c = _ctx(ctx)
    r, ln = C.c_double(), C.c_double()
    g = np.empty(F.shape + (3,)) if gradient else None
    c.check(c.lib.wlm_residual_lncc(c.h, _p(F), _p(M), _p(u), _dims(F.shape), int(radius),
                                    C.byref(r), C.byref(ln), _p(g) if gradient else None))
    return ResidualReport(r.value, g, ln.value)


def residual_mi(F, M, u, bins=32, sigma=1.0, gradient=True, ctx=None) -> ResidualReport:
    """residual_mi: r = log2(bins) - MI, loss_raw = MI (bits)."""
    F, M, u = _vol(F), _vol(M), _fld(u)
    if F.shape != M.shape or u.shape[:3] != F.shape:
        raise DimensionMismatch(2, "residual_mi: dimension mismatch")
    c = _ctx(ctx)
    r, mi = C.c_double(), C.c_double()
    g = np.empty(F.shape + (3,)) if gradient else None
    c.check(c.lib.wlm_residual_mi(c.h, _p(F), _p(M), _p(u), _dims(F.shape), int(bins), float(sigma),
                                  C.byref(r), C.byref(mi), _p(g) if gradient else None))
    return ResidualReport(r.value, g, mi.value)


def residual_mse(F, M, u, gradient=True, ctx=None) -> ResidualReport:
    """residual_mse: r = loss_raw = mean (f - m(x+u))^2."""
    F, M, u = _vol(F), _vol(M), _fld(u)
    if F.shape != M.shape or u.shape[:3] != F.shape:
        raise DimensionMismatch(2, "residual_mse: dimension mismatch")
    c = _ctx(ctx)
    r = C.c_double()
    g = np.empty(F.shape + (3,)) if gradient else None
    c.check(c.lib.wlm_residual_mse(c.h, _p(F), _p(M), _p(u), _dims(F.shape), C.byref(r),
                                   _p(g) if gradient else None))
    return ResidualReport(r.value, g, r.value)


def lm_step_tiled(r, g, lam, k, ctx=None):
    """lm_step_tiled (Eq. 5) on the GPU, fp64."""
    g = _fld(g)
    c = _ctx(ctx)
    out = np.empty_like(g)
    c.check(c.lib.wlm_lm_step_tiled(c.h, float(r), _p(g), _dims(g.shape), float(lam), int(k), _p(out)))
    return out


def demons_step_mse(r, n, alpha=1.0, ctx=None):
    """demons_step_mse (Eq. 9): r (nz,ny,nx) per-voxel residual,
    n (nz,ny,nx,3) moving gradient; returns the (nz,ny,nx,3) update."""
    r, n = _vol(r), _fld(n)
    if n.shape[:3] != r.shape:
        raise DimensionMismatch(2, "demons_step_mse: dimension mismatch")
    c = _ctx(ctx)
    out = np.empty_like(n)
    c.check(c.lib.wlm_demons_step_mse(c.h, _p(r), _p(n), _dims(r.shape), float(alpha), _p(out)))
    return out


def lm_step_pointwise(r, g, lam, ctx=None):
    g = _fld(g)
    c = _ctx(ctx)
    out = np.empty_like(g)
    c.check(c.lib.wlm_lm_step_pointwise(c.h, float(r), _p(g), _dims(g.shape), float(lam), _p(out)))
    return out


def lm_config(**kw) -> LmConfig:
    return reg_config(**{"lm." + k: v for k, v in kw.items()}).lm


def update_damping(state: LmState, loss_new, cfg: LmConfig) -> LmState:
    s = LmState(state.lam, state.hist_n, state.L1, state.L2)
    load().wlm_update_damping(C.byref(s), float(loss_new), C.byref(cfg))
    return s


def rejection_test(new, prev, prev2, tau=1.0) -> bool:
    return bool(load().wlm_rejection_test(float(new), float(prev), float(prev2), float(tau)))


def downsample(vol, factor, ctx=None):
    vol = _vol(vol)
    c = _ctx(ctx)
    f = int(factor)
    if f < 1:
        raise InvalidArgument(1, "downsample: factor < 1")
    shape = tuple(-(-n // f) for n in vol.shape)
    out = np.empty(shape)
    nd = Dims()
    c.check(c.lib.wlm_downsample(c.h, _p(vol), _dims(vol.shape), f, _p(out), C.byref(nd)))
    return out


def upsample_warp(u, new_shape, scale, ctx=None):
    u = _fld(u)
    c = _ctx(ctx)
    out = np.empty(tuple(new_shape) + (3,))
    c.check(c.lib.wlm_upsample_warp(c.h, _p(u), _dims(u.shape), _dims(new_shape), float(scale),
                                    _p(out)))
    return out


def synth_pair(shape, seed, num_blobs=12, warp_max=3.0, noise_sigma=0.01, warp_sigma=0.0, ctx=None):
    """synth_pair on the GPU: (fixed, moving, u_true) with
    shape (nz, ny, nx), u_true (nz, ny, nx, 3) AoS; moving is fixed sampled
    through Id + u_true.  Raises InvalidArgument when no positive-Jacobian
    warp is found in 10 draws."""
    from ._lib import SynthSpec
    nz, ny, nx = (int(s) for s in shape)
    c = _ctx(ctx)
    spec = SynthSpec(Dims(nx, ny, nz), int(num_blobs), float(warp_sigma), float(warp_max),
                     float(noise_sigma), int(seed))
    F = np.empty((nz, ny, nx), np.float32)
    M = np.empty_like(F)
    U = np.empty((3, nz, ny, nx), np.float32)
    c.check(c.lib.wlm_synth_pair(c.h, C.byref(spec), F.ctypes.data, M.ctypes.data, U.ctypes.data, 0))
    return F, M, np.ascontiguousarray(np.moveaxis(U, 0, -1))


def state_bytes(optimizer, shape, elem_bytes=4) -> int:
    return int(load().wlm_state_bytes(int(optimizer), _dims(shape), int(elem_bytes)))


def reg_config(**kw) -> RegConfig:
    """RegConfig with SPEC defaults; keys like 'lm.rejection', 'factors', 'iters'."""
    c = RegConfig()
    load().wlm_default_reg_config(C.byref(c))
    for k, v in kw.items():
        if k in ("factors", "iters"):
            arr = getattr(c, k)
            for i, x in enumerate(v):
                arr[i] = int(x)
        elif "." in k:
            a, b = k.split(".")
            setattr(getattr(c, a), b, v)
        else:
            setattr(c, k, v)
    return c


def trace_rows(rows):
    return [dict(level=t.level, iter=t.iter, loss_raw=t.loss_raw, r=t.r, lam=t.lam, eps=t.eps,
                 accepted=t.accepted, retries=t.retries, jac_det_min=t.jac_det_min) for t in rows]


def register(F, M, cfg: RegConfig | None = None, ctx=None) -> RegResult:
    """register(fixed, moving, RegConfig) -> RegResult."""
    cfg = cfg or reg_config()
    F = np.ascontiguousarray(F, dtype=np.float32)
    M = np.ascontiguousarray(M, dtype=np.float32)
    if F.shape != M.shape or F.ndim != 3:
        raise DimensionMismatch(2, "register: dimension mismatch")
    c = _ctx(ctx)
    warp = np.zeros(F.shape + (3,))
    cap = sum(cfg.iters[i] for i in range(cfg.nlevels)) + 1
    rows = (StepLog * cap)()
    n = C.c_size_t(0)
    jac = C.c_double(float("nan"))
    st = c.lib.wlm_register(c.h, F.ctypes.data_as(C.POINTER(C.c_float)),
                            M.ctypes.data_as(C.POINTER(C.c_float)), _dims(F.shape), C.byref(cfg),
                            _p(warp), rows, cap, C.byref(n), C.byref(jac))
    trace = [rows[i] for i in range(n.value)]
    if st != 0:
        err = WlmError if st != 3 else NonFiniteLoss
        e = err(st, c.lib.wlm_last_error(c.h).decode())
        e.partial_trace = trace
        raise e
    return RegResult(warp, trace, jac.value, c.peak_bytes)
