"""Host logic of the z-slab decomposition (config 5), no GPU needed:
partition, halo plan consistency, and the multi-process bootstrap over a
world_size-2/4 gloo group (what each rank would execute with NCCL)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_19371_b200 as P
from paper_2603_19371_b200 import slabs


def test_partition_covers_volume():
    for nz, ns in ((1024, 8), (1023, 8), (20, 5), (37, 3), (8, 2)):
        parts = slabs.partition(nz, ns)
        assert parts[0][0] == 0 and parts[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert all(ze - zs >= 4 for zs, ze in parts)
    with pytest.raises(ValueError):
        slabs.partition(12, 4)


def _halo_depths(cfg):
    import math
    r = lambda s: 0 if s <= 0 else max(1, math.ceil(3 * s))  # noqa: E731  field.cpp:206-207
    return dict(g=r(cfg.sigma_update), dU_s=r(cfg.sigma_warp), warp=max(r(cfg.sigma_warp) + 1, 2), abe=2)


def check_plans(shape, ns, plans, cfg):
    """Every receive has the matching send on the peer (same buffer, planes);
    sends come from owned planes; receives cover exactly the halo each
    stage reads (clipped at the volume faces)."""
    parts = slabs.partition(shape[0], ns)
    depth = _halo_depths(cfg)
    for k, rows in enumerate(plans):
        zs, ze = parts[k]
        for r in rows:
            peer = plans[r["peer"]]
            twin = [q for q in peer if q["peer"] == k and q["buffer"] == r["buffer"]
                    and q["send"] != r["send"] and (q["z0"], q["z1"]) == (r["z0"], r["z1"])]
            assert len(twin) == 1, (k, r)
            if r["send"]:
                assert zs <= r["z0"] < r["z1"] <= ze
            else:
                pz0, pz1 = parts[r["peer"]]
                assert pz0 <= r["z0"] < r["z1"] <= pz1 and not (zs <= r["z0"] < ze)
        for buf, h in depth.items():
            recv = sorted((r["z0"], r["z1"]) for r in rows if r["buffer"] == buf and not r["send"])
            want = [x for x in ((max(0, zs - h), zs), (ze, min(shape[0], ze + h))) if x[1] > x[0]]
            assert recv == want, (k, buf, recv, want)


@pytest.mark.parametrize("ns", [2, 3, 5, 8])
def test_halo_plans_match_pairwise(ns):
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[1])
    shape = (64, 16, 16)
    plans = [slabs.halo_plan(shape, ns, k, cfg) for k in range(ns)]
    check_plans(shape, ns, plans, cfg)


@pytest.mark.parametrize("ns", [2, 3, 5, 8])
@pytest.mark.parametrize("sig", [(1.0, 0.5), (0.5, 1.0), (2.0, 1.6)])
def test_fused_store_ranges_are_one_face_run_per_neighbour(ns, sig):
    """What the fused halo stores rely on (slab.cu setup_fused): per buffer
    kind a slab sends at most one row to each neighbour, the lower one's
    starting at its first owned plane and the upper one's ending at its
    last, so a producer's store test is 'plane < lo_end' / 'plane >=
    hi_begin'; and every send row's planes are exactly the receiver's halo
    rows of that kind (no plane the receiver itself writes)."""
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[1], sigma_update=sig[0], sigma_warp=sig[1])
    shape = (8 * ns + 16, 8, 8)
    parts = slabs.partition(shape[0], ns)
    plans = [slabs.halo_plan(shape, ns, k, cfg) for k in range(ns)]
    for k, rows in enumerate(plans):
        zs, ze = parts[k]
        for buf in ("g", "dU_s", "warp", "abe"):
            sends = [r for r in rows if r["buffer"] == buf and r["send"]]
            lo = [r for r in sends if r["peer"] == k - 1]
            hi = [r for r in sends if r["peer"] == k + 1]
            assert len(lo) == (1 if k > 0 else 0) and len(hi) == (1 if k + 1 < ns else 0)
            assert len(lo) + len(hi) == len(sends)
            if lo:
                assert lo[0]["z0"] == zs
                pz0, pz1 = parts[k - 1]
                assert not (pz0 <= lo[0]["z0"] < pz1)  # the receiver's halo, not its own planes
            if hi:
                assert hi[0]["z1"] == ze
                pz0, pz1 = parts[k + 1]
                assert not (pz0 <= hi[0]["z1"] - 1 < pz1)


def test_halo_plan_follows_sigma():
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[1], sigma_update=0.5, sigma_warp=1.0)
    shape = (40, 8, 8)
    plans = [slabs.halo_plan(shape, 4, k, cfg) for k in range(4)]
    check_plans(shape, 4, plans, cfg)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, shape, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.reg_config(nlevels=1, factors=[1], iters=[1])
        # the NCCL id travels from rank 0 exactly as RankSlab's bootstrap does
        uid = slabs.broadcast_unique_id(lambda: bytes(range(128)) if rank == 0 else None)
        mine = slabs.halo_plan(shape, world, rank, cfg)
        plans = [None] * world
        dist.all_gather_object(plans, mine)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        if rank == 0:
            check_plans(shape, world, plans, cfg)
            assert all(i == bytes(range(128)) for i in ids)
            q.put("ok")
    except Exception as e:  # surfaced by the parent
        q.put(f"rank {rank}: {e!r}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_bootstrap_and_plan_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, (48, 12, 10), q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == "ok"


def test_tiled_plans_have_twin_sends():
    """Tiled LM: slab boundaries on tile boundaries, the step matrices of the
    halo tiles travel as whole tile-planes; every receive has its twin send."""
    for k, ns in ((2, 3), (3, 2), (4, 3)):
        cfg = P.reg_config(nlevels=1, factors=[1], iters=[1], **{"lm.tile_size": k})
        shape = (40, 12, 10)
        plans = [slabs.halo_plan(shape, ns, s, cfg) for s in range(ns)]
        for s, rows in enumerate(plans):
            tm = [r for r in rows if r["buffer"] == "tm"]
            assert tm or ns == 1
            for r in tm:
                assert r["z0"] % k == 0 and (r["z1"] % k == 0 or r["z1"] == shape[0])
                twin = [q for q in plans[r["peer"]] if q["peer"] == s and q["buffer"] == "tm"
                        and q["send"] != r["send"] and (q["z0"], q["z1"]) == (r["z0"], r["z1"])]
                assert len(twin) == 1, (k, ns, s, r)


def test_halo_plan_refuses_what_a_group_refuses():
    """wlm_slab_halo_plan applies the slab group's own per-slab test: with
    tiles (k = 4) a split whose tile-aligned slabs are thinner than R_u + k
    is refused by both, though nz / nslabs alone would pass."""
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[1], **{"lm.tile_size": 4})
    with pytest.raises(ValueError):
        slabs.halo_plan((24, 8, 8), 4, 0, cfg)   # 6 planes per slab < R_u (3) + k (4)
    slabs.halo_plan((24, 8, 8), 3, 0, cfg)       # 8 planes per slab: fine


def test_nccl_shim_exports_what_the_transport_binds():
    """tests/nccl_shim/libnccl_shim.so (the two-rank stand-in of
    tests/test_slab_ranks.py) exports every symbol slab.cu's NCCL loader
    resolves, and hands out distinct unique ids (no GPU needed)."""
    import ctypes as C
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2603_19371_b200", "csrc", "slab.cu")).read()
    wanted = re.findall(r'SYM\(\w+, "(nccl\w+)"\)', src)
    assert len(wanted) >= 9
    lib = C.CDLL(os.path.join(root, "tests", "nccl_shim", "libnccl_shim.so"))
    assert all(hasattr(lib, w) for w in wanted), [w for w in wanted if not hasattr(lib, w)]
    a, b = C.create_string_buffer(128), C.create_string_buffer(128)
    assert lib.ncclGetUniqueId(a) == 0 and lib.ncclGetUniqueId(b) == 0 and a.raw != b.raw
