"""Device-resident batched LM engine (wlm_engine_* in include/wlm.h).

A batch of independent registrations of identical dims stays in HBM; one
``step()`` is one lm_iterate attempt for every pair (K2 gradient, K3 LM step
+ smoothing + max, K4 compositive resample + smoothing, K1 warp + LNCC +
device-side damping/rejection), captured as a CUDA graph.  Inputs may be
host numpy arrays or device pointers (e.g. ``torch.Tensor.data_ptr()``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Dims, LmState, RegConfig, StepLog, load
from .warplm import _LIVE_ENGINES, Context, default_context, reg_config, trace_rows


class Engine:
    def __init__(self, shape, pairs=1, cfg: RegConfig | None = None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.lib = load()
        self.shape = tuple(int(s) for s in shape)  # (nz, ny, nx)
        self.pairs = int(pairs)
        self.cfg = cfg or reg_config()
        nz, ny, nx = self.shape
        h = C.c_void_p()
        self.ctx.check(self.lib.wlm_engine_create(self.ctx.h, Dims(nx, ny, nz), self.pairs,
                                                  C.byref(self.cfg), C.byref(h)))
        self.h = h
        _LIVE_ENGINES.add(self)

    @property
    def nvox(self):
        nz, ny, nx = self.shape
        return nx * ny * nz

    def _chk(self, st):
        self.ctx.check(st)

    @staticmethod
    def _ptr(a):
        """(pointer, is_host) for a numpy array or a CUDA tensor / int pointer."""
        if isinstance(a, np.ndarray):
            return a.ctypes.data, 1
        if hasattr(a, "data_ptr"):
            return a.data_ptr(), 0 if a.is_cuda else 1
        return int(a), 0

    def load(self, F, M):
        """F, M: (pairs, nz, ny, nx) float32 (host numpy or device tensor)."""
        if isinstance(F, np.ndarray):
            F = np.ascontiguousarray(F, dtype=np.float32)
            M = np.ascontiguousarray(M, dtype=np.float32)
        pf, hf = self._ptr(F)
        pm, _ = self._ptr(M)
        self._keep = (F, M)
        self._chk(self.lib.wlm_engine_load(self.h, pf, pm, hf))

    def set_warp(self, u=None):
        """u: (pairs, 3, nz, ny, nx) float32 SoA or None for the identity."""
        if u is None:
            self._chk(self.lib.wlm_engine_set_warp(self.h, None, 1))
            return
        if isinstance(u, np.ndarray):
            u = np.ascontiguousarray(u, dtype=np.float32)
        p, host = self._ptr(u)
        self._chk(self.lib.wlm_engine_set_warp(self.h, p, host))
        self.ctx.synchronize()

    def get_warp(self):
        out = np.empty((self.pairs, 3) + self.shape, np.float32)
        self._chk(self.lib.wlm_engine_get_warp(self.h, out.ctypes.data, 1))
        return out

    def get_warp_device(self, tensor):
        self._chk(self.lib.wlm_engine_get_warp(self.h, tensor.data_ptr(), 0))

    def reset(self):
        """New registrations on the loaded pairs: lambda back to lambda0
        (begin_level alone carries lambda, as between pyramid levels)."""
        self._chk(self.lib.wlm_engine_reset(self.h))

    def begin_level(self, level=0):
        self._chk(self.lib.wlm_engine_begin_level(self.h, int(level)))

    def iterate(self, iters):
        self._chk(self.lib.wlm_engine_iterate(self.h, int(iters)))

    def set_pair_groups(self, groups):
        """1..4 independent streams of attempt graphs in iterate() (wlm.h)."""
        self._chk(self.lib.wlm_engine_set_pair_groups(self.h, int(groups)))

    def step(self):
        self._chk(self.lib.wlm_engine_step(self.h))

    def state(self, pair=0):
        st = LmState()
        r, ln = C.c_double(), C.c_double()
        it = C.c_int()
        self._chk(self.lib.wlm_engine_state(self.h, pair, C.byref(st), C.byref(r), C.byref(ln),
                                            C.byref(it)))
        return dict(lam=st.lam, hist_n=st.hist_n, L1=st.L1, L2=st.L2, r=r.value, lncc=ln.value,
                    iters=it.value)

    def trace(self, pair=0, cap=100000):
        rows = (StepLog * cap)()
        n = C.c_size_t()
        self._chk(self.lib.wlm_engine_trace(self.h, pair, rows, cap, C.byref(n)))
        return trace_rows(rows[i] for i in range(n.value))

    def buffers(self):
        ptrs = [C.c_void_p() for _ in range(6)]
        self._chk(self.lib.wlm_engine_buffers(self.h, *[C.byref(p) for p in ptrs]))
        return dict(zip(("F", "M", "u", "g", "vs", "abe"), (p.value for p in ptrs)))

    BUF = {"F": 0, "M": 1, "u": 2, "g": 3, "vs": 4, "abe": 5}

    def read_buffer(self, name, pair=0):
        """Host copy of one pair's engine buffer (F, M: (nz,ny,nx); u, g, vs,
        abe: (3,nz,ny,nx)) -- test / debug hook."""
        nch = 1 if name in ("F", "M") else 4 if name == "abe" else 3
        out = np.empty((nch,) + self.shape, np.float32)
        self._chk(self.lib.wlm_engine_read_buffer(self.h, self.BUF[name], pair, out.ctypes.data,
                                                  out.size))
        if name == "abe":  # A, B fp32 planes + E fp64 plane
            return out[0], out[1], out[2:].reshape(-1).view(np.float64).reshape(self.shape)
        return out[0] if nch == 1 else out

    def script_losses(self, losses):
        """losses: (pairs, n) float64 -- scripted-residual harness."""
        if losses is None:
            self._chk(self.lib.wlm_engine_script_losses(self.h, None, 0))
            return
        a = np.ascontiguousarray(losses, dtype=np.float64).reshape(self.pairs, -1)
        self._chk(self.lib.wlm_engine_script_losses(self.h, a.ctypes.data_as(C.POINTER(C.c_double)),
                                                    a.shape[1]))

    def close(self):
        if getattr(self, "h", None):
            self.lib.wlm_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SlabGroup:
    """One registration split into ``nslabs`` z-slabs (wlm_slab_group_* in
    include/wlm.h, config 5).  Same calls as :class:`Engine` with pairs = 1;
    results are bit-identical for every ``nslabs``."""

    def __init__(self, shape, nslabs, cfg: RegConfig | None = None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.lib = load()
        self.shape = tuple(int(s) for s in shape)
        self.nslabs = int(nslabs)
        self.cfg = cfg or reg_config()
        nz, ny, nx = self.shape
        h = C.c_void_p()
        self.ctx.check(self.lib.wlm_slab_group_create(self.ctx.h, Dims(nx, ny, nz), self.nslabs,
                                                      C.byref(self.cfg), C.byref(h)))
        self.h = h
        _LIVE_ENGINES.add(self)

    def _chk(self, st):
        self.ctx.check(st)

    def load(self, F, M):
        """F, M: whole (nz, ny, nx) float32 volumes (numpy or CUDA tensor)."""
        if isinstance(F, np.ndarray):
            F = np.ascontiguousarray(F, dtype=np.float32)
            M = np.ascontiguousarray(M, dtype=np.float32)
        pf, hf = Engine._ptr(F)
        pm, _ = Engine._ptr(M)
        self._chk(self.lib.wlm_slab_group_load(self.h, pf, pm, hf))
        self.ctx.synchronize()

    def set_warp(self, u=None):
        if u is None:
            self._chk(self.lib.wlm_slab_group_set_warp(self.h, None, 1))
            return
        if isinstance(u, np.ndarray):
            u = np.ascontiguousarray(u, dtype=np.float32)
        p, host = Engine._ptr(u)
        self._chk(self.lib.wlm_slab_group_set_warp(self.h, p, host))

    def get_warp(self, out=None):
        """Whole-volume (3, nz, ny, nx) warp (planes owned elsewhere are left
        untouched); out may be a numpy array or a pinned/CUDA tensor."""
        if out is None:
            out = np.zeros((3,) + self.shape, np.float32)
        p, host = Engine._ptr(out)
        self._chk(self.lib.wlm_slab_group_get_warp(self.h, p, host))
        return out

    def begin_level(self, level=0):
        self._chk(self.lib.wlm_slab_group_begin_level(self.h, int(level)))

    def reset(self):
        """New registration: lambda back to lambda0 (begin_level carries it)."""
        self._chk(self.lib.wlm_slab_group_reset(self.h))

    def fused_halos(self):
        """Bit mask of the halo exchanges fused into their producing kernels
        (bit 0 g, 1 dU_s, 2 warp, 3 A/B/E; include/wlm.h)."""
        m = C.c_int()
        self._chk(self.lib.wlm_slab_group_fused_halos(self.h, C.byref(m)))
        return m.value

    def iterate(self, iters):
        self._chk(self.lib.wlm_slab_group_iterate(self.h, int(iters)))

    def state(self):
        st = LmState()
        r, ln = C.c_double(), C.c_double()
        it = C.c_int()
        self._chk(self.lib.wlm_slab_group_state(self.h, C.byref(st), C.byref(r), C.byref(ln),
                                                C.byref(it)))
        return dict(lam=st.lam, hist_n=st.hist_n, L1=st.L1, L2=st.L2, r=r.value, lncc=ln.value,
                    iters=it.value)

    def trace(self, cap=100000):
        rows = (StepLog * cap)()
        n = C.c_size_t()
        self._chk(self.lib.wlm_slab_group_trace(self.h, rows, cap, C.byref(n)))
        return trace_rows(rows[i] for i in range(n.value))

    def close(self):
        if getattr(self, "h", None):
            self.lib.wlm_slab_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BatchPipeline:
    """Serving loop for a stream of batches of identical geometry: two engines
    (two contexts, two streams) alternate, so batch k+1's input copy and
    batch k's warp copy run under the other engine's iterations.  Each batch
    is one registration level of ``iters`` iterations from the identity warp
    (the bench's pipelined e2e measurement is this loop).

        pipe = BatchPipeline((192, 192, 192), pairs=8, cfg=cfg, iters=100)
        for warps in pipe.run(batches):   # batches: iterable of (F, M)
            ...                            # (pairs, 3, nz, ny, nx) float32

    Results are those of running every batch alone on one engine.  Inputs
    may be host arrays (pinned memory overlaps best) or CUDA tensors."""

    def __init__(self, shape, pairs, cfg: RegConfig | None = None, iters=100, device=0):
        self.shape = tuple(int(s) for s in shape)
        self.pairs = int(pairs)
        self.iters = int(iters)
        self.ctxs = [Context(device), Context(device)]
        self.engines = [Engine(self.shape, self.pairs, cfg, ctx=c) for c in self.ctxs]

    def _launch(self, eng, F, M):
        eng.load(F, M)
        eng.set_warp(None)
        eng.reset()  # a new batch is a new registration: lambda0, not the last batch's lambda
        eng.begin_level(0)
        eng.iterate(self.iters)

    def run(self, batches):
        pending = None
        for k, (F, M) in enumerate(batches):
            eng = self.engines[k % 2]
            self._launch(eng, F, M)      # queued behind nothing on this engine's stream
            if pending is not None:
                yield pending.get_warp()  # the other engine: waits for its iterations, copies out
            pending = eng
        if pending is not None:
            yield pending.get_warp()

    def close(self):
        for e in self.engines:
            e.close()
        for c in self.ctxs:
            c.close()
