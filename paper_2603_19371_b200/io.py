"""VOL3 / DSP3 files and the CSV trace (reference io.hpp:15-21).

Host reads/writes run without a GPU (pure host path of the C ABI); pass a
CUDA tensor to read straight into device memory (streamed through pinned
staging) or to write a device-resident warp.  Every reference ``io_error``
raises :class:`IoError` with the reference's message.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import Dims, InvalidArgument, StepLog, load
from .warplm import Context, default_context

__all__ = ["IoError", "read_vol3", "write_vol3", "read_dsp3", "write_dsp3", "write_trace_csv",
           "register_files"]


class IoError(InvalidArgument):
    """warplm::io_error (io.hpp:11-13)."""


def _err(ctx, status, what):
    msg = ctx.lib.wlm_last_error(ctx.h).decode() if ctx is not None else what
    raise IoError(status, msg)


def _dims(path, field):
    d = Dims()
    st = load().wlm_io_dims(os.fsencode(path), 1 if field else 0, C.byref(d))
    if st != 0:
        raise IoError(st, f"{path}: unreadable {'DSP3' if field else 'VOL3'} header")
    return d


def read_vol3(path, out=None, ctx: Context | None = None):
    """(nz, ny, nx) float32.  ``out``: optional CUDA tensor (device read)."""
    lib = load()
    d = _dims(path, False)
    shape = (d.nz, d.ny, d.nx)
    got = Dims()
    if out is None:
        arr = np.empty(shape, np.float32)
        st = lib.wlm_read_vol3(None, os.fsencode(path), arr.ctypes.data, arr.size, 0, C.byref(got))
        if st != 0:
            raise IoError(st, f"{path}: malformed VOL3")
        return arr
    ctx = ctx or default_context()
    st = lib.wlm_read_vol3(ctx.h, os.fsencode(path), out.data_ptr(), out.numel(), 1, C.byref(got))
    if st != 0:
        _err(ctx, st, path)
    return out


def write_vol3(path, vol, ctx: Context | None = None):
    lib = load()
    if hasattr(vol, "is_cuda") and vol.is_cuda:
        ctx = ctx or default_context()
        nz, ny, nx = vol.shape
        st = lib.wlm_write_vol3(ctx.h, os.fsencode(path), vol.data_ptr(), 1, Dims(nx, ny, nz))
        if st != 0:
            _err(ctx, st, path)
        return
    a = np.ascontiguousarray(vol, dtype=np.float32)
    nz, ny, nx = a.shape
    st = lib.wlm_write_vol3(None, os.fsencode(path), a.ctypes.data, 0, Dims(nx, ny, nz))
    if st != 0:
        raise IoError(st, f"{path}: write failed")


def read_dsp3(path, out=None, ctx: Context | None = None):
    """SoA (3, nz, ny, nx) float32 (the engine layout).  ``out``: optional CUDA
    tensor; the AoS payload is transposed on the device."""
    lib = load()
    d = _dims(path, True)
    shape = (3, d.nz, d.ny, d.nx)
    got = Dims()
    if out is None:
        arr = np.empty(shape, np.float32)
        st = lib.wlm_read_dsp3(None, os.fsencode(path), arr.ctypes.data, arr.size, 0, C.byref(got))
        if st != 0:
            raise IoError(st, f"{path}: malformed DSP3")
        return arr
    ctx = ctx or default_context()
    st = lib.wlm_read_dsp3(ctx.h, os.fsencode(path), out.data_ptr(), out.numel(), 1, C.byref(got))
    if st != 0:
        _err(ctx, st, path)
    return out


def write_dsp3(path, u_soa, ctx: Context | None = None):
    """u_soa: (3, nz, ny, nx) float32 (numpy or CUDA tensor)."""
    lib = load()
    if hasattr(u_soa, "is_cuda") and u_soa.is_cuda:
        ctx = ctx or default_context()
        _, nz, ny, nx = u_soa.shape
        st = lib.wlm_write_dsp3(ctx.h, os.fsencode(path), u_soa.data_ptr(), 1, Dims(nx, ny, nz))
        if st != 0:
            _err(ctx, st, path)
        return
    a = np.ascontiguousarray(u_soa, dtype=np.float32)
    _, nz, ny, nx = a.shape
    st = lib.wlm_write_dsp3(None, os.fsencode(path), a.ctypes.data, 0, Dims(nx, ny, nz))
    if st != 0:
        raise IoError(st, f"{path}: write failed")


def write_trace_csv(path, trace):
    """trace: RegResult.loss_trace rows (StepLog structs, or dicts with the
    SPEC.md:427 keys as Engine.trace returns them)."""
    rows = (StepLog * max(1, len(trace)))()
    for i, t in enumerate(trace):
        if isinstance(t, StepLog):
            rows[i] = t
        else:
            rows[i] = StepLog(t["level"], t["iter"], t["loss_raw"], t["r"], t["lam"], t["eps"], t["accepted"],
                              t["retries"], t["jac_det_min"])
    st = load().wlm_write_trace_csv(os.fsencode(path), rows, len(trace))
    if st != 0:
        raise IoError(st, f"{path}: write failed")


def register_files(fixed_path, moving_path, warp_path, csv_path=None, cfg=None, ctx=None):
    """cmd_register semantics as an API: VOL3 in, DSP3 warp
    and CSV trace out; returns the RegResult."""
    from .warplm import register
    F = read_vol3(fixed_path)
    M = read_vol3(moving_path)
    if F.shape != M.shape:
        raise IoError(2, f"{fixed_path}, {moving_path}: dimension mismatch")
    res = register(F, M, cfg, ctx=ctx)
    write_dsp3(warp_path, np.ascontiguousarray(np.moveaxis(res.final_warp, -1, 0), dtype=np.float32))
    if csv_path:
        write_trace_csv(csv_path, res.loss_trace)
    return res
