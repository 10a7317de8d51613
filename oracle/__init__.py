"""TEST INFRASTRUCTURE ONLY -- ctypes bindings onto the fp64 CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2603_19371_b200`` never imports it and has no CPU fallback.

Two shared objects (built by oracle/Makefile):
  liboracle.so          self-contained fp64 restatement (see oracle.h)
  _ref/liboracle_ref.so same spec-only modules on top of the unmodified
                        reference field.cpp/io.cpp, plus ref_* entry points
                        onto the raw reference functions.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "liboracle_ref.so")

MAX_LEVELS = 8
OPT_LM, OPT_ADAM, OPT_GD = 0, 1, 2


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int)]


class LmConfig(C.Structure):
    _fields_ = [("lambda0", C.c_double), ("mu_plus", C.c_double), ("mu_minus", C.c_double),
                ("tile_size", C.c_int), ("rejection", C.c_int), ("tau", C.c_double),
                ("lambda_max", C.c_double), ("max_retries", C.c_int)]


class LmState(C.Structure):
    _fields_ = [("lam", C.c_double), ("hist_n", C.c_int), ("L1", C.c_double),
                ("L2", C.c_double)]


class AdamConfig(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps_hat", C.c_double),
                ("lr", C.c_double)]


class RegConfig(C.Structure):
    _fields_ = [("lncc_radius", C.c_int), ("optimizer", C.c_int), ("lm", LmConfig),
                ("adam", AdamConfig), ("gd_lr", C.c_double), ("nlevels", C.c_int),
                ("factors", C.c_int * MAX_LEVELS), ("iters", C.c_int * MAX_LEVELS),
                ("target_max_disp", C.c_double), ("step_floor", C.c_double),
                ("sigma_update", C.c_double), ("sigma_warp", C.c_double),
                ("log_jacobian", C.c_int), ("metric", C.c_int), ("demons_alpha", C.c_double),
                ("mi_bins", C.c_int), ("mi_sigma", C.c_double)]


class StepLog(C.Structure):
    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("loss_raw", C.c_double),
                ("r", C.c_double), ("lam", C.c_double), ("eps", C.c_double),
                ("accepted", C.c_int), ("retries", C.c_int), ("jac_det_min", C.c_double)]


class SynthSpec(C.Structure):
    _fields_ = [("dims", Dims), ("num_blobs", C.c_int), ("warp_sigma", C.c_double),
                ("warp_max", C.c_double), ("noise_sigma", C.c_double), ("seed", C.c_uint64)]


_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I = C.POINTER(C.c_int)


def _p(a, t=_D):
    return None if a is None else a.ctypes.data_as(t)


def _declare(lib):
    sig = {
        "orc_set_threads": (None, [C.c_int]),
        "orc_set_fp32_storage": (None, [C.c_int]),
        "orc_set_dev_flags": (None, [C.c_int]),
        "orc_dev_smooth32": (None, [_D, Dims, C.c_double, C.c_int]),
        "orc_default_reg_config": (None, [C.POINTER(RegConfig)]),
        "orc_sample_trilinear_grad": (C.c_double, [_D, Dims, C.c_double, C.c_double, C.c_double, _D]),
        "orc_sample_field": (None, [_D, Dims, C.c_double, C.c_double, C.c_double, _D]),
        "orc_warp_volume": (None, [_D, _D, Dims, _D, _D]),
        "orc_compose_warp": (None, [_D, _D, Dims, C.c_double, _D]),
        "orc_max_abs_component": (C.c_double, [_D, C.c_size_t]),
        "orc_normalize_step": (C.c_double, [_D, C.c_size_t, C.c_double, C.c_double]),
        "orc_jacobian_det_min": (C.c_double, [_D, Dims]),
        "orc_gaussian_smooth": (None, [_D, Dims, C.c_int, C.c_double]),
        "orc_all_finite": (C.c_int, [_D, C.c_size_t]),
        "orc_residual_lncc": (C.c_double, [_D, _D, _D, Dims, C.c_int, _D, _D, _D]),
        "orc_residual_mse": (C.c_double, [_D, _D, _D, Dims, _D]),
        "orc_residual_mi": (C.c_double, [_D, _D, _D, Dims, C.c_int, C.c_double, _D, _D]),
        "orc_demons_step_mse": (None, [_D, _D, C.c_size_t, C.c_double, _D]),
        "orc_lm_step_pointwise": (None, [C.c_double, _D, C.c_size_t, C.c_double, _D]),
        "orc_lm_step_dense3": (None, [C.c_double, _D, C.c_double, _D]),
        "orc_lm_step_tiled": (None, [C.c_double, _D, Dims, C.c_double, C.c_int, _D]),
        "orc_update_damping": (None, [C.POINTER(LmState), C.c_double, C.POINTER(LmConfig)]),
        "orc_rejection_test": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double]),
        "orc_lm_replay": (C.c_int, [_D, C.c_int, C.c_int, C.POINTER(LmConfig), _D, _I,
                                    C.POINTER(LmState)]),
        "orc_adam_step": (None, [_D, _D, _D, C.c_size_t, C.c_int, C.POINTER(AdamConfig), _D]),
        "orc_level_dims": (Dims, [Dims, C.c_int]),
        "orc_downsample": (None, [_D, Dims, C.c_int, _D]),
        "orc_upsample_warp": (None, [_D, Dims, Dims, C.c_double, _D]),
        "orc_lm_run_level": (C.c_int, [_D, _D, Dims, _D, C.POINTER(RegConfig), C.POINTER(LmState),
                                       C.c_int, C.c_int, C.POINTER(StepLog), _I]),
        "orc_lm_run_level_timed": (C.c_int, [_D, _D, Dims, _D, C.POINTER(RegConfig), C.POINTER(LmState),
                                             C.c_int, C.c_int, C.POINTER(StepLog), _I, _D, C.c_int, _I]),
        "orc_register": (C.c_int, [_F, _F, Dims, C.POINTER(RegConfig), _D, C.POINTER(StepLog),
                                   C.c_size_t, C.POINTER(C.c_size_t), _D]),
        "orc_synth_pair": (C.c_int, [C.POINTER(SynthSpec), _F, _F, _F]),
        "orc_splitmix64": (C.c_uint64, [C.POINTER(C.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_libs: dict = {}


def lib(kind: str = "port"):
    """kind 'port' -> liboracle.so; 'reference' -> _ref/liboracle_ref.so."""
    if kind not in _libs:
        path = LIB_PATH if kind == "port" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        L = _declare(C.CDLL(path))
        L.orc_set_threads(min(8, os.cpu_count() or 1))
        _libs[kind] = L
    return _libs[kind]


class fp32_storage:
    """Context manager: run the oracle with device storage-precision emulation."""

    def __init__(self, kind="port", mode=1):
        self.kind, self.mode = kind, mode

    def __enter__(self):
        lib(self.kind).orc_set_fp32_storage(self.mode)
        return self

    def __exit__(self, *a):
        lib(self.kind).orc_set_fp32_storage(0)


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def ref_lib():
    """The raw reference functions (ref_* symbols) in _ref/liboracle_ref.so."""
    L = lib("reference")
    if not getattr(L, "_ref_declared", False):
        L.ref_sample_trilinear_grad.restype = C.c_double
        L.ref_sample_trilinear_grad.argtypes = [_D, C.c_int, C.c_int, C.c_int, C.c_double,
                                                C.c_double, C.c_double, _D]
        L.ref_warp_volume.argtypes = [_D, _D, C.c_int, C.c_int, C.c_int, _D, _D]
        L.ref_sample_field.argtypes = [_D, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, _D]
        L.ref_compose_warp.restype = C.c_int
        L.ref_compose_warp.argtypes = [_D, C.c_int, C.c_int, C.c_int, _D, C.c_int, C.c_int,
                                       C.c_int, C.c_double, _D]
        L.ref_max_abs_component.restype = C.c_double
        L.ref_max_abs_component.argtypes = [_D, C.c_int, C.c_int, C.c_int]
        L.ref_normalize_step.restype = C.c_double
        L.ref_normalize_step.argtypes = [_D, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double]
        L.ref_jacobian_det_min.restype = C.c_double
        L.ref_jacobian_det_min.argtypes = [_D, C.c_int, C.c_int, C.c_int]
        L.ref_gaussian_smooth.argtypes = [_D, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
        L.ref_all_finite.restype = C.c_int
        L.ref_all_finite.argtypes = [_D, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_write_vol3.restype = C.c_int
        L.ref_write_vol3.argtypes = [C.c_char_p, _D, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.ref_write_dsp3.restype = C.c_int
        L.ref_write_dsp3.argtypes = [C.c_char_p, _D, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.ref_read.restype = C.c_int
        L.ref_read.argtypes = [C.c_char_p, C.c_int, _I, _D, C.c_size_t, C.c_char_p, C.c_int]
        L._ref_declared = True
    return L


# ---------------------------------------------------------------------------
# numpy-facing helpers.  Volumes are (nz, ny, nx) float64 C-contiguous arrays
# (x fastest, reference Dims3::index); fields are (nz, ny, nx, 3) (AoS,
# component innermost, reference DispField3).

def dims_of(a) -> Dims:
    return Dims(a.shape[2], a.shape[1], a.shape[0])


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_config(**kw) -> RegConfig:
    c = RegConfig()
    lib().orc_default_reg_config(C.byref(c))
    for k, v in kw.items():
        if k in ("factors", "iters"):
            arr = getattr(c, k)
            for i, x in enumerate(v):
                arr[i] = x
        elif "." in k:
            a, b = k.split(".")
            setattr(getattr(c, a), b, v)
        else:
            setattr(c, k, v)
    return c


def sample_trilinear_grad(vol, p, kind="port"):
    vol = _c64(vol)
    g = np.zeros(3)
    v = lib(kind).orc_sample_trilinear_grad(_p(vol), dims_of(vol), float(p[0]), float(p[1]),
                                            float(p[2]), _p(g))
    return v, g


def warp_volume(M, u, kind="port"):
    M, u = _c64(M), _c64(u)
    Mw = np.empty_like(M)
    gM = np.empty(M.shape + (3,))
    lib(kind).orc_warp_volume(_p(M), _p(u), dims_of(M), _p(Mw), _p(gM))
    return Mw, gM


def compose_warp(u, v, eps, kind="port"):
    u, v = _c64(u), _c64(v)
    out = np.empty_like(u)
    lib(kind).orc_compose_warp(_p(u), _p(v), dims_of(u), float(eps), _p(out))
    return out


def max_abs_component(v, kind="port"):
    v = _c64(v)
    return lib(kind).orc_max_abs_component(_p(v), v.size)


def normalize_step(v, target=0.4, floor=1e-12, kind="port"):
    v = _c64(v)
    return lib(kind).orc_normalize_step(_p(v), v.size, target, floor)


def jacobian_det_min(u, kind="port"):
    u = _c64(u)
    return lib(kind).orc_jacobian_det_min(_p(u), dims_of(u))


def gaussian_smooth(a, sigma, kind="port"):
    out = _c64(a).copy()
    nch = 3 if out.ndim == 4 else 1
    lib(kind).orc_gaussian_smooth(_p(out), dims_of(out), nch, float(sigma))
    return out


@dataclass
class LnccInternals:
    Mw: np.ndarray
    rho: np.ndarray
    A: np.ndarray
    B: np.ndarray
    E: np.ndarray
    dMw: np.ndarray
    gradM: np.ndarray


def residual_lncc(F, M, u, radius=2, internals=False, kind="port"):
    F, M, u = _c64(F), _c64(M), _c64(u)
    g = np.empty(F.shape + (3,))
    ln = C.c_double()
    N = F.size
    it = np.empty(9 * N) if internals else None
    r = lib(kind).orc_residual_lncc(_p(F), _p(M), _p(u), dims_of(F), radius, _p(g),
                                    C.byref(ln), _p(it))
    if internals:
        s = F.shape
        ins = LnccInternals(it[:N].reshape(s), it[N:2 * N].reshape(s), it[2 * N:3 * N].reshape(s),
                            it[3 * N:4 * N].reshape(s), it[4 * N:5 * N].reshape(s),
                            it[5 * N:6 * N].reshape(s), it[6 * N:].reshape(s + (3,)))
        return r, g, ln.value, ins
    return r, g, ln.value


def residual_mi(F, M, u, bins=32, sigma=1.0, kind="port"):
    """(r, g, MI): r = log2(bins) - MI in bits."""
    F, M, u = _c64(F), _c64(M), _c64(u)
    g = np.empty(F.shape + (3,))
    mi = C.c_double()
    r = lib(kind).orc_residual_mi(_p(F), _p(M), _p(u), dims_of(F), int(bins), float(sigma), _p(g),
                                  C.byref(mi))
    return r, g, mi.value


def residual_mse(F, M, u, kind="port"):
    F, M, u = _c64(F), _c64(M), _c64(u)
    g = np.empty(F.shape + (3,))
    r = lib(kind).orc_residual_mse(_p(F), _p(M), _p(u), dims_of(F), _p(g))
    return r, g


def demons_step_mse(r, n, alpha, kind="port"):
    r, n = _c64(r), _c64(n)
    out = np.empty_like(n)
    lib(kind).orc_demons_step_mse(_p(r), _p(n), r.size, float(alpha), _p(out))
    return out


def lm_step_pointwise(r, g, lam, kind="port"):
    g = _c64(g)
    out = np.empty_like(g)
    lib(kind).orc_lm_step_pointwise(float(r), _p(g), g.size // 3, float(lam), _p(out))
    return out


def lm_step_tiled(r, g, lam, k, kind="port"):
    g = _c64(g)
    out = np.empty_like(g)
    lib(kind).orc_lm_step_tiled(float(r), _p(g), dims_of(g[..., 0]), float(lam), int(k), _p(out))
    return out


def lm_step_dense3(r, g3, lam):
    g3 = _c64(g3)
    out = np.empty(3)
    lib().orc_lm_step_dense3(float(r), _p(g3), float(lam), _p(out))
    return out


def lm_config(**kw) -> LmConfig:
    return default_config(**{"lm." + k: v for k, v in kw.items()}).lm


def update_damping(state: LmState, loss_new, cfg: LmConfig) -> LmState:
    s = LmState(state.lam, state.hist_n, state.L1, state.L2)
    lib().orc_update_damping(C.byref(s), float(loss_new), C.byref(cfg))
    return s


def rejection_test(new, prev, prev2, tau=1.0) -> bool:
    return bool(lib().orc_rejection_test(float(new), float(prev), float(prev2), float(tau)))


def lm_replay(losses, iters, cfg: LmConfig, state: LmState | None = None):
    losses = _c64(losses)
    n = losses.size
    lam = np.zeros(n)
    dec = np.zeros(n, dtype=np.int32)
    st = state or LmState(cfg.lambda0, 0, 0.0, 0.0)
    k = lib().orc_lm_replay(_p(losses), n, iters, C.byref(cfg), _p(lam), _p(dec, _I), C.byref(st))
    return lam[:k], dec[:k], st


def adam_step(g, m, v, t, lr=0.5, beta1=0.9, beta2=0.999, eps_hat=1e-8):
    g = _c64(g)
    out = np.empty_like(g)
    c = AdamConfig(beta1, beta2, eps_hat, lr)
    lib().orc_adam_step(_p(g), _p(m), _p(v), g.size, int(t), C.byref(c), _p(out))
    return out


def level_dims(shape, f):
    d = lib().orc_level_dims(Dims(shape[2], shape[1], shape[0]), int(f))
    return (d.nz, d.ny, d.nx)


def downsample(vol, f, kind="port"):
    vol = _c64(vol)
    out = np.empty(level_dims(vol.shape, f))
    lib(kind).orc_downsample(_p(vol), dims_of(vol), int(f), _p(out))
    return out


def upsample_warp(u, new_shape, scale, kind="port"):
    u = _c64(u)
    out = np.empty(tuple(new_shape) + (3,))
    nd = Dims(new_shape[2], new_shape[1], new_shape[0])
    lib(kind).orc_upsample_warp(_p(u), Dims(u.shape[2], u.shape[1], u.shape[0]), nd,
                                float(scale), _p(out))
    return out


def lm_run_level(F, M, u, cfg: RegConfig, iters, state: LmState | None = None, level=0,
                 kind="port"):
    F, M = _c64(F), _c64(M)
    u = _c64(u).copy()
    st = state or LmState(cfg.lm.lambda0, 0, 0.0, 0.0)
    trace = (StepLog * max(iters, 1))()
    nt = C.c_int(0)
    rc = lib(kind).orc_lm_run_level(_p(F), _p(M), dims_of(F), _p(u), C.byref(cfg), C.byref(st),
                                    level, iters, trace, C.byref(nt))
    return rc, u, st, [trace[i] for i in range(nt.value)]


def lm_run_level_timed(F, M, u, cfg: RegConfig, iters, kind="port"):
    """lm_run_level plus the wall time of every attempt (LM step through the
    residual at the trial warp; the level's initial residual excluded)."""
    F, M = _c64(F), _c64(M)
    u = _c64(u).copy()
    st = LmState(cfg.lm.lambda0, 0, 0.0, 0.0)
    trace = (StepLog * max(iters, 1))()
    nt = C.c_int(0)
    cap = max(1, iters * (cfg.lm.max_retries + 1))
    times = np.zeros(cap)
    na = C.c_int(0)
    rc = lib(kind).orc_lm_run_level_timed(_p(F), _p(M), dims_of(F), _p(u), C.byref(cfg), C.byref(st),
                                          0, iters, trace, C.byref(nt), _p(times), cap, C.byref(na))
    return rc, u, [trace[i] for i in range(nt.value)], times[:na.value]


def register(F, M, cfg: RegConfig, kind="port"):
    F = np.ascontiguousarray(F, dtype=np.float32)
    M = np.ascontiguousarray(M, dtype=np.float32)
    warp = np.zeros(F.shape + (3,))
    cap = sum(cfg.iters[i] for i in range(cfg.nlevels)) + 1
    trace = (StepLog * cap)()
    n = C.c_size_t(0)
    jac = C.c_double(0.0)
    rc = lib(kind).orc_register(_p(F, _F), _p(M, _F), dims_of(F), C.byref(cfg), _p(warp), trace,
                                cap, C.byref(n), C.byref(jac))
    return rc, warp, [trace[i] for i in range(n.value)], jac.value


def synth_pair(shape, seed, num_blobs=12, warp_max=3.0, noise_sigma=0.01, warp_sigma=0.0):
    """Returns (F, M, u_true) as float32 arrays; shape = (nz, ny, nx)."""
    nz, ny, nx = shape
    s = SynthSpec(Dims(nx, ny, nz), num_blobs, warp_sigma, warp_max, noise_sigma, seed)
    F = np.empty(shape, np.float32)
    M = np.empty(shape, np.float32)
    U = np.empty(tuple(shape) + (3,), np.float32)
    rc = lib().orc_synth_pair(C.byref(s), _p(F, _F), _p(M, _F), _p(U, _F))
    if rc != 0:
        raise ValueError("synth_pair: no positive-Jacobian warp after 10 draws")
    return F, M, U


def trace_rows(trace):
    return [dict(level=t.level, iter=t.iter, loss_raw=t.loss_raw, r=t.r, lam=t.lam, eps=t.eps,
                 accepted=t.accepted, retries=t.retries, jac_det_min=t.jac_det_min) for t in trace]
