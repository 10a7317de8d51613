"""z-slab decomposition of one registration (config 5).

Host side of wlm_slab_* (include/wlm.h): the partition and halo plan (pure
host logic, usable without a GPU), the in-process slab group and the
one-process-per-GPU form, whose NCCL communicator is bootstrapped over any
torch.distributed process group (the 128-byte NCCL unique id is broadcast
from rank 0 as a uint8 tensor, so gloo works too).
"""
from __future__ import annotations

import ctypes as C
import glob
import os

import numpy as np

from ._lib import Dims, HaloXfer, RegConfig, load
from .engine import SlabGroup
from .warplm import Context, default_context, reg_config

BUFFERS = ("g", "dU_s", "warp", "abe", "tm")


def partition(nz, nslabs):
    """[(zs, ze)] owned planes of every slab (raises if a slab < 4 planes)."""
    lib = load()
    out = []
    for k in range(nslabs):
        zs, ze = C.c_int(), C.c_int()
        st = lib.wlm_slab_partition(int(nz), int(nslabs), k, C.byref(zs), C.byref(ze))
        if st != 0:
            raise ValueError(f"cannot split {nz} planes into {nslabs} slabs of >= 4 planes")
        out.append((zs.value, ze.value))
    return out


def halo_plan(shape, nslabs, slab, cfg: RegConfig | None = None):
    """Exchange rows of one slab: dicts (buffer, peer, send, z0, z1)."""
    lib = load()
    cfg = cfg or reg_config()
    nz, ny, nx = shape
    n = C.c_size_t()
    d = Dims(nx, ny, nz)
    st = lib.wlm_slab_halo_plan(d, nslabs, slab, C.byref(cfg), None, 0, C.byref(n))
    if st != 0:
        raise ValueError("invalid slab split")
    rows = (HaloXfer * max(1, n.value))()
    lib.wlm_slab_halo_plan(d, nslabs, slab, C.byref(cfg), C.cast(rows, C.c_void_p), n.value, C.byref(n))
    return [dict(buffer=BUFFERS[r.buffer], peer=r.peer, send=bool(r.send), z0=r.z0, z1=r.z1)
            for r in rows[:n.value]]


def nccl_library():
    """Path of the libnccl.so.2 to dlopen: $WLM_NCCL_LIB when set (e.g. the
    two-rank test stand-in), else the one torch uses, or None."""
    env = os.environ.get("WLM_NCCL_LIB")
    if env:
        return env
    try:
        import nvidia.nccl  # noqa: F401
        for d in nvidia.nccl.__path__:
            hits = glob.glob(os.path.join(d, "lib", "libnccl.so*"))
            if hits:
                return sorted(hits)[0]
    except ImportError:
        pass
    return None


def broadcast_unique_id(make_id, group=None):
    """Rank 0 calls make_id() -> 128 bytes; every rank returns those bytes.
    Works over gloo (CPU tensor) and nccl (moved to the current device)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        raw = make_id()
        assert len(raw) == 128
        buf = torch.frombuffer(bytearray(raw), dtype=torch.uint8).clone()
    backend = dist.get_backend(group)
    if backend == "nccl":
        dev = buf.cuda()
        dist.broadcast(dev, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        buf = dev.cpu()
    else:
        dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group else 0, group=group)
    return bytes(buf.numpy().tobytes())


def nccl_unique_id(lib_path=None):
    lib = load()
    out = C.create_string_buffer(128)
    st = lib.wlm_nccl_unique_id((lib_path or nccl_library() or "").encode(), out)
    if st != 0:
        raise RuntimeError(f"ncclGetUniqueId failed (status {st})")
    return out.raw[:128]


class RankSlab(SlabGroup):
    """Slab ``rank`` of ``nranks`` held by this process (one GPU per rank).
    Collective calls (create, begin_level, iterate) must be made by every
    rank in the same order."""

    def __init__(self, shape, rank, nranks, uid: bytes, cfg: RegConfig | None = None,
                 ctx: Context | None = None, nccl_lib=None):
        self.ctx = ctx or default_context()
        self.lib = load()
        self.shape = tuple(int(s) for s in shape)
        self.nslabs = int(nranks)
        self.rank = int(rank)
        self.cfg = cfg or reg_config()
        nz, ny, nx = self.shape
        h = C.c_void_p()
        path = (nccl_lib or nccl_library() or "").encode()
        self.ctx.check(self.lib.wlm_slab_group_create_nccl(
            self.ctx.h, Dims(nx, ny, nz), self.rank, self.nslabs, bytes(uid), path,
            C.byref(self.cfg), C.byref(h)))
        self.h = h
        from .warplm import _LIVE_ENGINES
        _LIVE_ENGINES.add(self)

    def owned(self):
        zs, ze = C.c_int(), C.c_int()
        self._chk(self.lib.wlm_slab_group_owned(self.h, C.byref(zs), C.byref(ze)))
        return zs.value, ze.value

    def get_local_warp(self):
        """(3, ze - zs, ny, nx) owned planes of the accepted warp."""
        zs, ze = self.owned()
        full = self.get_warp()
        return np.ascontiguousarray(full[:, zs:ze])
