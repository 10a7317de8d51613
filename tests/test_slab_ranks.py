"""Config 5's distributed data plane with 2, 3 and 4 ranks (VERDICT r1 "next" #6).

The one-process-per-GPU slab transport (csrc/slab.cu, wlm_slab_group_create_nccl)
runs as one process per slab, each holding one z-slab, exchanging halo rows with
ncclSend/ncclRecv and all-reducing the per-plane sum(rho) (foreign planes
zeroed), max |dU_s|, min det J and MI histograms.  This box has one GPU, so the
ranks share it and the NCCL library the transport dlopens is the test
stand-in tests/nccl_shim/libnccl_shim.so (the same ABI over CUDA IPC with
host-side synchronisation: no kernel of one rank waits on the other's).

Bar: every rank's trace and the owned planes of its warp are bit-identical
to the single-domain engine's, with and without rejection (whose retry loop
re-reads the device state on the host), with Adam, and with MI; with the
fused halo stores (K2, K3, K4 and K1b store the neighbour's halo planes
into its buffer, mapped by CUDA IPC, and the exchange is a 4-byte ordering
token) and with the copy exchange.
"""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SHIM = os.path.join(HERE, "nccl_shim", "libnccl_shim.so")

pytestmark = pytest.mark.gpu

SHAPE = (24, 20, 28)  # (nz, ny, nx): two slabs of 12 planes
CASES = [{}, {"lm.rejection": 1, "lm.tau": 0.05, "log_jacobian": 1}, {"optimizer": 1}, {"metric": 2},
         {"low_memory": 1}]


def _pair():
    import oracle as O
    F, M, _ = O.synth_pair(SHAPE, 23, num_blobs=8, warp_max=2.5)
    return F, M


def _rank(rank, uid, extra, iters, q, nranks=2):
    sys.path.insert(0, ROOT)
    try:
        import paper_2603_19371_b200 as P
        from paper_2603_19371_b200 import slabs
        F, M = _pair()
        ctx = P.Context(0)
        cfg = P.reg_config(nlevels=1, factors=[1], iters=[iters], **extra)
        grp = slabs.RankSlab(SHAPE, rank, nranks, uid, cfg=cfg, ctx=ctx, nccl_lib=SHIM)
        fused = grp.fused_halos()
        grp.load(F, M)
        grp.set_warp(None)
        grp.begin_level(0)
        grp.iterate(iters)
        zs, ze = grp.owned()
        q.put((rank, zs, ze, grp.get_local_warp(), grp.trace(), grp.state(), fused))
        grp.close()
        ctx.close()
    except Exception as e:  # report, never hang the parent
        q.put((rank, "error", repr(e)))


def _unique_id():
    import ctypes as C
    lib = C.CDLL(SHIM)
    buf = C.create_string_buffer(128)
    assert lib.ncclGetUniqueId(buf) == 0
    return buf.raw[:128]


def same_trace(a, b):
    return len(a) == len(b) and all(
        all((x[k] == y[k]) or (x[k] != x[k] and y[k] != y[k]) for k in x) for x, y in zip(a, b))


def _single_domain(P, ctx, extra, iters):
    F, M = _pair()
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[iters], **extra)
    eng = P.Engine(SHAPE, pairs=1, cfg=cfg, ctx=ctx)
    eng.load(F[None], M[None])
    eng.set_warp(None)
    eng.begin_level(0)
    eng.iterate(iters)
    out = eng.get_warp()[0], eng.trace(0), eng.state(0)
    eng.close()
    return out


def _run_ranks(nranks, extra, iters):
    uid = _unique_id()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    ps = [mpc.Process(target=_rank, args=(r, uid, extra, iters, q, nranks)) for r in range(nranks)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(nranks):
        item = q.get(timeout=300)
        assert item[1] != "error", item
        got[item[0]] = item
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("nranks,extra", [(3, {}), (4, {"lm.rejection": 1, "lm.tau": 0.05, "log_jacobian": 1}),
                                          (4, {"optimizer": 1})])
def test_three_and_four_rank_slabs_bit_identical(ctx, nranks, extra):
    """Middle ranks (two neighbours: sends and receives on both faces in one
    group) through the same transport: 3 and 4 processes, bit-identical to
    the single domain."""
    import paper_2603_19371_b200 as P
    iters = 20
    w1, t1, s1 = _single_domain(P, ctx, extra, iters)
    got = _run_ranks(nranks, extra, iters)
    z = 0
    for r in range(nranks):
        _, zs, ze, w, t, s, fm = got[r]
        assert fm == (0b1111 if extra.get("optimizer", 0) != 1 else 0b1110), fm
        assert zs == z and ze > zs
        z = ze
        assert same_trace(t, t1), (r, extra)
        assert s["lam"] == s1["lam"] and s["r"] == s1["r"]
        assert np.array_equal(w, w1[:, zs:ze]), (r, float(np.abs(w - w1[:, zs:ze]).max()))
    assert z == SHAPE[0]


@pytest.mark.parametrize("extra", CASES)
@pytest.mark.parametrize("fused", ["1", "0"])
def test_two_rank_slabs_bit_identical_to_single_domain(ctx, extra, fused, monkeypatch):
    """Two ranks, with the producers' fused halo stores into the
    neighbour's buffer mapped by CUDA IPC (default) and with the NCCL
    send/recv copy exchange (WLM_SLAB_FUSED=0); the spawned ranks inherit
    the setting."""
    monkeypatch.setenv("WLM_SLAB_FUSED", fused)
    import paper_2603_19371_b200 as P
    assert os.path.exists(SHIM), "build the shim: make (tests/nccl_shim/libnccl_shim.so)"
    iters = 20  # with rejection (tau 0.05) the oracle retries 20 times on this pair
    w1, t1, s1 = _single_domain(P, ctx, extra, iters)
    got = _run_ranks(2, extra, iters)
    owned = []
    want = 0 if fused == "0" else (0b1110 if extra.get("optimizer", 0) == 1 else
                                   0b0110 if extra.get("metric", 0) != 0 else 0b1111)
    for r in range(2):
        _, zs, ze, w, t, s, fm = got[r]
        assert fm == want, (fm, want)
        owned.append((zs, ze))
        assert same_trace(t, t1), (r, extra)
        assert s["lam"] == s1["lam"] and s["r"] == s1["r"]
        assert np.array_equal(w, w1[:, zs:ze]), (r, float(np.abs(w - w1[:, zs:ze]).max()))
    assert owned == [(0, 12), (12, 24)]
    if extra.get("lm.rejection"):
        assert sum(row["retries"] for row in t1) > 0, "the case should exercise the retry loop"


@pytest.mark.parametrize("nproc,size", [(2, 96), (4, 128)])
def test_bench_config5_ranks_under_torchrun(nproc, size):
    """bench.py --config 5 under the driver's torchrun launch with two and
    four ranks (one GPU: gloo for torch.distributed, the NCCL stand-in for
    the slab transport via WLM_NCCL_LIB; four ranks have middle slabs with
    two neighbours): one JSON line from rank 0, strong scaling, the slab
    group's multi-rank path (unique-id broadcast, RankSlab, owned planes,
    fused halo stores, e2e with host buffers) end to end."""
    import json
    import subprocess
    env = dict(os.environ, WLM_BENCH_BACKEND="gloo", WLM_NCCL_LIB=SHIM)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
                          "--master-addr", "127.0.0.1", "--master-port", str(29541 + nproc),
                          os.path.join(ROOT, "bench.py"), "--config", "5", "--size", str(size), "--gpus", str(nproc),
                          "--steps", "3", "--warmup", "3", "--e2e-iters", "2"],
                         capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == nproc and line["scaling"] == "strong" and line["value"] > 0
    assert f"z-slab x{nproc}" in line["config"]["parallelism"] and line["e2e"]["value"] > 0
    assert line["config"]["fused_halos"] == "1111"  # every exchange fused into its producer
