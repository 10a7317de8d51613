"""ctypes binding of the C-ABI (include/wlm.h) of libwarplm_b200.so.

The shared library is built in-tree by ``make`` (see __graft_entry__.build).
There is no fallback: if the library is missing or no CUDA device is
visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# WLM_LIB_PATH selects another build of the same library (A/B kernel variants)
LIB_PATH = os.environ.get("WLM_LIB_PATH") or os.path.join(HERE, "libwarplm_b200.so")

MAX_LEVELS = 8
OPT_LM, OPT_ADAM, OPT_GD, OPT_DEMONS = 0, 1, 2, 3
METRIC_LNCC, METRIC_MSE, METRIC_MI = 0, 1, 2

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "DIM_MISMATCH", 3: "NONFINITE", 4: "OOM", 5: "CUDA",
          6: "UNSUPPORTED"}


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int)]


class LmConfig(C.Structure):
    _fields_ = [("lambda0", C.c_double), ("mu_plus", C.c_double), ("mu_minus", C.c_double),
                ("tile_size", C.c_int), ("rejection", C.c_int), ("tau", C.c_double),
                ("lambda_max", C.c_double), ("max_retries", C.c_int)]


class LmState(C.Structure):
    _fields_ = [("lam", C.c_double), ("hist_n", C.c_int), ("L1", C.c_double), ("L2", C.c_double)]


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
                ("mi_bins", C.c_int), ("mi_sigma", C.c_double), ("low_memory", C.c_int)]


class SynthSpec(C.Structure):
    _fields_ = [("dims", Dims), ("num_blobs", C.c_int), ("warp_sigma", C.c_double),
                ("warp_max", C.c_double), ("noise_sigma", C.c_double), ("seed", C.c_uint64)]


class HaloXfer(C.Structure):
    _fields_ = [("buffer", C.c_int), ("peer", C.c_int), ("send", C.c_int), ("z0", C.c_int),
                ("z1", C.c_int)]


class StepLog(C.Structure):
    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("loss_raw", C.c_double),
                ("r", C.c_double), ("lam", C.c_double), ("eps", C.c_double),
                ("accepted", C.c_int), ("retries", C.c_int), ("jac_det_min", C.c_double)]


_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_VP = C.c_void_p
_CTX = C.c_void_p
_ENG = C.c_void_p

# name -> (restype, argtypes).  Every symbol declared in include/wlm.h.
SIGNATURES = {
    "wlm_ctx_create": (C.c_int, [C.c_int, C.POINTER(_CTX)]),
    "wlm_ctx_destroy": (None, [_CTX]),
    "wlm_last_error": (C.c_char_p, [_CTX]),
    "wlm_ctx_stream": (_VP, [_CTX]),
    "wlm_ctx_set_stream": (C.c_int, [_CTX, _VP]),
    "wlm_ctx_synchronize": (C.c_int, [_CTX]),
    "wlm_ctx_launch_count": (C.c_uint64, [_CTX]),
    "wlm_default_reg_config": (None, [C.POINTER(RegConfig)]),
    "wlm_version": (C.c_char_p, []),
    "wlm_source_hash": (C.c_char_p, []),
    "wlm_warp_volume": (C.c_int, [_CTX, _D, _D, Dims, _D, _D]),
    "wlm_sample_field_points": (C.c_int, [_CTX, _D, Dims, _D, C.c_size_t, _D]),
    "wlm_sample_trilinear_grad_points": (C.c_int, [_CTX, _D, Dims, _D, C.c_size_t, _D, _D]),
    "wlm_compose_warp": (C.c_int, [_CTX, _D, Dims, _D, Dims, C.c_double, _D]),
    "wlm_max_abs_component": (C.c_int, [_CTX, _D, Dims, _D]),
    "wlm_normalize_step": (C.c_int, [_CTX, _D, Dims, C.c_double, C.c_double, _D]),
    "wlm_jacobian_det_min": (C.c_int, [_CTX, _D, Dims, _D]),
    "wlm_gaussian_smooth_vol": (C.c_int, [_CTX, _D, Dims, C.c_double, _D]),
    "wlm_gaussian_smooth_field": (C.c_int, [_CTX, _D, Dims, C.c_double, _D]),
    "wlm_all_finite": (C.c_int, [_CTX, _D, C.c_size_t, C.POINTER(C.c_int)]),
    "wlm_residual_lncc": (C.c_int, [_CTX, _D, _D, _D, Dims, C.c_int, _D, _D, _D]),
    "wlm_residual_mse": (C.c_int, [_CTX, _D, _D, _D, Dims, _D, _D]),
    "wlm_residual_mi": (C.c_int, [_CTX, _D, _D, _D, Dims, C.c_int, C.c_double, _D, _D, _D]),
    "wlm_demons_step_mse": (C.c_int, [_CTX, _D, _D, Dims, C.c_double, _D]),
    "wlm_lm_step_tiled": (C.c_int, [_CTX, C.c_double, _D, Dims, C.c_double, C.c_int, _D]),
    "wlm_lm_step_pointwise": (C.c_int, [_CTX, C.c_double, _D, Dims, C.c_double, _D]),
    "wlm_update_damping": (None, [C.POINTER(LmState), C.c_double, C.POINTER(LmConfig)]),
    "wlm_rejection_test": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double]),
    "wlm_downsample": (C.c_int, [_CTX, _D, Dims, C.c_int, _D, C.POINTER(Dims)]),
    "wlm_upsample_warp": (C.c_int, [_CTX, _D, Dims, Dims, C.c_double, _D]),
    "wlm_state_bytes": (C.c_size_t, [C.c_int, Dims, C.c_int]),
    "wlm_register": (C.c_int, [_CTX, _F, _F, Dims, C.POINTER(RegConfig), _D, C.POINTER(StepLog),
                               C.c_size_t, C.POINTER(C.c_size_t), _D]),
    "wlm_ctx_peak_bytes": (C.c_size_t, [_CTX]),
    "wlm_engine_create": (C.c_int, [_CTX, Dims, C.c_int, C.POINTER(RegConfig), C.POINTER(_ENG)]),
    "wlm_engine_destroy": (None, [_ENG]),
    "wlm_engine_load": (C.c_int, [_ENG, _VP, _VP, C.c_int]),
    "wlm_engine_set_warp": (C.c_int, [_ENG, _VP, C.c_int]),
    "wlm_engine_get_warp": (C.c_int, [_ENG, _VP, C.c_int]),
    "wlm_engine_begin_level": (C.c_int, [_ENG, C.c_int]),
    "wlm_engine_iterate": (C.c_int, [_ENG, C.c_int]),
    "wlm_engine_set_pair_groups": (C.c_int, [_ENG, C.c_int]),
    "wlm_engine_reset": (C.c_int, [_ENG]),
    "wlm_engine_step": (C.c_int, [_ENG]),
    "wlm_engine_state": (C.c_int, [_ENG, C.c_int, C.POINTER(LmState), _D, _D,
                                   C.POINTER(C.c_int)]),
    "wlm_engine_trace": (C.c_int, [_ENG, C.c_int, C.POINTER(StepLog), C.c_size_t,
                                   C.POINTER(C.c_size_t)]),
    "wlm_engine_buffers": (C.c_int, [_ENG, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP),
                                     C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP)]),
    "wlm_engine_script_losses": (C.c_int, [_ENG, _D, C.c_int]),
    "wlm_engine_stage": (C.c_int, [_ENG, C.c_int]),
    "wlm_engine_read_buffer": (C.c_int, [_ENG, C.c_int, C.c_int, _VP, C.c_size_t]),
    "wlm_slab_partition": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]),
    "wlm_slab_halo_plan": (C.c_int, [Dims, C.c_int, C.c_int, C.POINTER(RegConfig), _VP, C.c_size_t,
                                     C.POINTER(C.c_size_t)]),
    "wlm_slab_group_create": (C.c_int, [_CTX, Dims, C.c_int, C.POINTER(RegConfig), C.POINTER(_ENG)]),
    "wlm_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_char_p]),
    "wlm_slab_group_create_nccl": (C.c_int, [_CTX, Dims, C.c_int, C.c_int, C.c_char_p, C.c_char_p,
                                             C.POINTER(RegConfig), C.POINTER(_ENG)]),
    "wlm_slab_group_owned": (C.c_int, [_ENG, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "wlm_slab_group_fused_halos": (C.c_int, [_ENG, C.POINTER(C.c_int)]),
    "wlm_slab_group_destroy": (None, [_ENG]),
    "wlm_slab_group_load": (C.c_int, [_ENG, _VP, _VP, C.c_int]),
    "wlm_slab_group_set_warp": (C.c_int, [_ENG, _VP, C.c_int]),
    "wlm_slab_group_get_warp": (C.c_int, [_ENG, _VP, C.c_int]),
    "wlm_slab_group_begin_level": (C.c_int, [_ENG, C.c_int]),
    "wlm_slab_group_reset": (C.c_int, [_ENG]),
    "wlm_slab_group_iterate": (C.c_int, [_ENG, C.c_int]),
    "wlm_slab_group_trace": (C.c_int, [_ENG, C.POINTER(StepLog), C.c_size_t, C.POINTER(C.c_size_t)]),
    "wlm_slab_group_state": (C.c_int, [_ENG, C.POINTER(LmState), _D, _D, C.POINTER(C.c_int)]),
    "wlm_io_dims": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(Dims)]),
    "wlm_read_vol3": (C.c_int, [_CTX, C.c_char_p, _VP, C.c_size_t, C.c_int, C.POINTER(Dims)]),
    "wlm_read_dsp3": (C.c_int, [_CTX, C.c_char_p, _VP, C.c_size_t, C.c_int, C.POINTER(Dims)]),
    "wlm_write_vol3": (C.c_int, [_CTX, C.c_char_p, _VP, C.c_int, Dims]),
    "wlm_write_dsp3": (C.c_int, [_CTX, C.c_char_p, _VP, C.c_int, Dims]),
    "wlm_write_trace_csv": (C.c_int, [C.c_char_p, C.POINTER(StepLog), C.c_size_t]),
    "wlm_synth_pair": (C.c_int, [_CTX, C.POINTER(SynthSpec), _VP, _VP, _VP, C.c_int]),
}

_lib = None


def source_hash():
    """sha256 (16 hex digits) of the sources the Makefile hashes into the
    library, in the same (sorted path) order; None if they are absent."""
    import glob
    import hashlib
    root = os.path.dirname(HERE)
    rels = [os.path.relpath(p, root) for p in glob.glob(os.path.join(HERE, "csrc", "*.cu"))
            + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))] + [os.path.join("include", "wlm.h")]
    paths = [os.path.join(root, r) for r in sorted(rels)]
    if not all(os.path.exists(p) for p in paths):
        return None
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def load():
    """Load libwarplm_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build())")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        want = source_hash()
        got = lib.wlm_source_hash().decode()
        if want is not None and got != want and not os.environ.get("WLM_LIB_PATH"):
            raise ImportError(f"{LIB_PATH} was built from other sources (hash {got}, sources {want}): "
                              "run `make` (or __graft_entry__.build())")
        _lib = lib
    return _lib


class WlmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class DimensionMismatch(WlmError, ValueError):
    pass


class InvalidArgument(WlmError, ValueError):
    pass


class NonFiniteLoss(WlmError, ArithmeticError):
    pass


def check(status, ctx=None):
    if status == 0:
        return
    msg = load().wlm_last_error(ctx).decode() if ctx else ""
    cls = {1: InvalidArgument, 2: DimensionMismatch, 3: NonFiniteLoss}.get(status, WlmError)
    raise cls(status, msg)
