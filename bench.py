"""Benchmark of the factored-LM iteration (BASELINE.json config 4).

Workload: config 4, a batch of 64 independent 192^3 synthetic pairs split
64/N per GPU (strong scaling: the global batch is fixed), LNCC + LM,
rejection off.  One step = one lm_iterate attempt for every pair on the GPU
(K2 gradient, K3 LM step + smoothing + max, K4 compositive resample +
smoothing, K1 warp + LNCC + device-side damping).  Inputs (~31 GB per GPU at
N=1) are far larger than L2, so no flush is needed.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python bench.py --cpu-tables     # + config-1 and 192^3 primitive CPU tables

Multi-GPU: launched by torchrun, one rank per GPU; no data-path collective
(pairs are independent); timing = max over ranks (NCCL all-reduce of the
per-rank CUDA-event time).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
# Algorithmic HBM bytes per voxel per kernel: SURVEY 8(d)'s canonical figures
# (each logical array read or written once per stage, fp32), the numerator of
# roofline.achieved:
#   K1 eval  : u 12 + F 4 + M 4 + write A, B, E 12                   = 32
#   K2 grad  : A, B, E 12 + F 4 + u 12 + M 4 + write g 12            = 44
#   K3 step  : g 12 + write dU_s 12                                  = 24
#   K4 comp. : dU_s 12 + u 12 + write u' 12                          = 36
# This design moves more by choice: E in fp64 (+4 B in
# K1 and K2), Mw in fp64 between K1a and K1b (+16 B), and grad M(x+u) in fp64
# from K1a to K2 instead of a second gather (+24 B write, +24 B read, -16 B
# u/M in K2) -- reported as design_bytes_per_voxel.
KERNEL_BYTES = {"K1_lncc_fwd": 32, "K2_lncc_bwd": 44, "K3_step_smooth": 24, "K4_compose_smooth": 36}
DESIGN_BYTES = {"K1_lncc_fwd": 76, "K2_lncc_bwd": 64, "K3_step_smooth": 24, "K4_compose_smooth": 36}
STAGE_ID = {"K1_lncc_fwd": 0, "K2_lncc_bwd": 1, "K3_step_smooth": 2, "K4_compose_smooth": 3}
BYTES_PER_VOXEL_ITER = sum(KERNEL_BYTES.values())  # 136 (SURVEY 8(d) canonical)


def config4(n, global_batch, world):
    """The `config` object of both arms (identical, so the driver's arms
    compare like with like); per-arm details live outside it."""
    return {"workload": f"config 4: batch of {global_batch} independent {n}^3 pairs, LNCC r=2 + "
                        f"pointwise LM, rejection off",
            "global_batch": global_batch, "volume": [n, n, n],
            "parallelism": f"dp{world} (independent pairs split {global_batch}/{world} per GPU, "
                           f"no collective)",
            "l2": f"inputs > L2 (68 B/voxel x {n ** 3} voxels per pair)"}


def warp_max(n):
    """Config 4's maximum displacement (6 voxels at 192^3), scaled down for
    the small sizes the tests use (a 6-voxel warp folds a 24^3 volume)."""
    return 6.0 if n >= 96 else n / 16.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    10 ms while the timed region runs (the B200_PROFILING.md clocks line)."""

    REASONS = {  # nvmlClocksEventReason* bits that reject / annotate a run
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index, period=0.01):
        self.index, self.period = index, period
        self.samples, self.masks = [], []
        self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        import pynvml
        h = self.h
        while not self._stop.is_set():
            try:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                self.masks.append(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # NVML unavailable: report it, never guess
            self.err = repr(e)
            self.t = None
        return self

    def __exit__(self, *a):
        if self.t:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        reasons = sorted({k for m in self.masks for k, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def dist_init(n_gpus):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch
        import torch.distributed as dist
        # WLM_BENCH_BACKEND=gloo exercises the multi-rank path on fewer GPUs
        # than ranks (host barrier and max; ranks share devices round-robin,
        # so the timings are not scaling numbers)
        if os.environ.get("WLM_BENCH_BACKEND", "nccl") == "gloo":
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def max_over_ranks(x, world, local):
    """Max of a per-rank scalar (NCCL: on the rank's device; gloo: host)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world, local):
    if world > 1:
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()


# ------------------------------------------------------------------ ours ----
def run_ours(args, rank, world, local):
    import ctypes as C

    import numpy as np
    import torch

    import paper_2603_19371_b200 as P
    from paper_2603_19371_b200._lib import Dims, SynthSpec

    torch.cuda.set_device(local)
    n = args.size
    shape = (n, n, n)
    nvox = n ** 3
    pairs = args.pairs_per_gpu or max(1, args.global_batch // world)
    ctx = P.Context(local)
    lib = P.load()
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[100], low_memory=args.low_memory)
    eng = P.Engine(shape, pairs=pairs, cfg=cfg, ctx=ctx)

    # synthetic pairs (config 4 seeds 1000..1063), generated on the GPU by the
    # product's own synth_pair into pinned host memory (the e2e inputs)
    F_h = torch.empty((pairs,) + shape, dtype=torch.float32, pin_memory=True)
    M_h = torch.empty((pairs,) + shape, dtype=torch.float32, pin_memory=True)
    for p in range(pairs):
        seed = 1000 + rank * pairs + p
        spec = SynthSpec(Dims(n, n, n), 12, 0.0, warp_max(n), 0.01, seed)
        ctx.check(lib.wlm_synth_pair(ctx.h, C.byref(spec), F_h[p].data_ptr(), M_h[p].data_ptr(),
                                     None, 0))
    stream = torch.cuda.ExternalStream(ctx.stream(), device=f"cuda:{local}")

    eng.load(F_h, M_h)
    eng.set_warp(None)
    eng.begin_level(0)
    launches0 = ctx.launches
    eng.iterate(args.warmup)
    ctx.synchronize()

    # ---- device-resident throughput (value) ----
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(world, local)
    torch.cuda.synchronize()
    launches_before = ctx.launches
    with ClockSampler(local) as clk:
        ev0.record(stream)
        eng.iterate(args.steps)  # K attempts of every pair (rejection off), one call
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(world, local)
    launches_timed = ctx.launches - launches_before
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world, local)
    st = eng.state(0)
    assert math.isfinite(st["r"]) and st["iters"] == args.warmup + args.steps, st
    eng.begin_level(0)  # pairs reached their targets: re-arm them for the per-stage timing

    # ---- per-kernel durations (same stream, CUDA events around each launch) ----
    per_kernel = {}
    reps = max(3, min(10, args.steps))
    for name, sid in STAGE_ID.items():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        # keep the engine state coherent: run whole attempts, time one stage
        for a, b in evs:
            for other in (1, 2, 3, 0):
                if other == sid:
                    a.record(stream)
                    ctx.check(lib.wlm_engine_stage(eng.h, other))
                    b.record(stream)
                else:
                    ctx.check(lib.wlm_engine_stage(eng.h, other))
        torch.cuda.synchronize()
        per_kernel[name] = statistics.median(a.elapsed_time(b) for a, b in evs)
    hbm, peak_kind = peaks()
    dom = max(per_kernel, key=per_kernel.get)
    launch_vox = pairs * nvox
    achieved = KERNEL_BYTES[dom] * launch_vox / (per_kernel[dom] * 1e-3) / 1e9

    # ---- end to end through the C-ABI with host buffers (e2e) ----
    # per step: pinned host F, M -> device (wlm_engine_load), 100 LM
    # iterations (wlm_engine_iterate), accepted warps -> pinned host
    # (wlm_engine_get_warp).  Metric = voxel-iterations / time.
    e2e_iters = args.e2e_iters
    U_h = torch.empty((pairs, 3) + shape, dtype=torch.float32, pin_memory=True)

    def e2e_once():
        eng.load(F_h, M_h)
        eng.set_warp(None)
        eng.reset()
        eng.begin_level(0)
        eng.iterate(e2e_iters)
        ctx.check(lib.wlm_engine_get_warp(eng.h, U_h.data_ptr(), 1))

    e2e_once()  # warm (graph already built)
    e2e_steps = max(1, min(2, args.steps))
    barrier(world, local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    torch.cuda.synchronize()
    serial_s = max_over_ranks(time.perf_counter() - t0, world, local)
    serial_val = world * pairs * nvox * e2e_iters * e2e_steps / serial_s / 1e9

    # Pipelined: two engines (two contexts, two streams) alternate steps, so
    # step k+1's host->device input copy runs under step k's iterations and
    # step k's device->host warp copy under step k+1's.  Every step still
    # copies its inputs in and its warps out inside the timed region.
    ctx2 = P.Context(local)
    eng2 = P.Engine(shape, pairs=pairs, cfg=cfg, ctx=ctx2)
    engines = ((eng, ctx), (eng2, ctx2))
    for e, _ in engines:  # the two engines already overlap each other
        e.set_pair_groups(args.e2e_groups)

    def e2e_launch(e):
        e.load(F_h, M_h)
        e.set_warp(None)
        e.reset()  # each step registers its pairs afresh
        e.begin_level(0)
        e.iterate(e2e_iters)

    def e2e_finish(e, c):
        c.check(lib.wlm_engine_get_warp(e.h, U_h.data_ptr(), 1))

    for e, c in engines:  # warm the second engine's graph
        e2e_launch(e)
        e2e_finish(e, c)
    pipe_steps = max(2, min(4, args.steps))
    barrier(world, local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_launch(engines[0][0])
    for k in range(1, pipe_steps):
        e2e_launch(engines[k % 2][0])
        e2e_finish(*engines[(k - 1) % 2])
    e2e_finish(*engines[(pipe_steps - 1) % 2])
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world, local)
    e2e_val = world * pairs * nvox * e2e_iters * pipe_steps / e2e_s / 1e9
    eng2.close()
    ctx2.close()
    assert np.isfinite(U_h[0, :, ::17, ::17, ::17].numpy()).all()

    value = world * pairs * nvox * args.steps / (ms_max * 1e-3) / 1e9  # Gvoxel/s
    iters_per_s = world * pairs * args.steps / (ms_max * 1e-3)
    it_frac = BYTES_PER_VOXEL_ITER * value * 1e9 / (hbm * 1e9)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample([(F_h[p].numpy(), M_h[p].numpy()) for p in range(pairs)])
        if args.cpu_tables:
            cpu["tables"] = cpu_tables()
    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        eng.close()  # free the batch engine before the pyramid runs
        extra = pyramid_configs(ctx, lib)

    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "Gvoxel/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 5),
        "higher_is_better": True,
        "scaling": "strong" if not args.pairs_per_gpu else "weak",
        "vs_baseline": None,
        "dtype": "f64", "storage_dtype": "f32",
        "data": "synthetic (GPU synth_pair: Gaussian blobs + smoothed random warp max 6, noise 0.01, "
                "seeds 1000+)",
        "config": config4(n, world * pairs, world),
        "pairs_per_gpu": pairs,
        "iters_per_s": round(iters_per_s, 2),
        "iters_per_s_per_pair": round(args.steps / (ms_max * 1e-3), 2),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                     "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": None,
                     "algorithmic_bytes_per_voxel": KERNEL_BYTES[dom],
                     "design_bytes_per_voxel": DESIGN_BYTES[dom],
                     "per_kernel_ms": {k: round(v, 4) for k, v in per_kernel.items()},
                     # every stage against the same peak: canonical bytes / time
                     "per_kernel_frac": {k: round(KERNEL_BYTES[k] * launch_vox / (v * 1e-3) / 1e9 / hbm, 4)
                                         for k, v in per_kernel.items()},
                     "per_kernel_traffic": {k: load_traffic(k) for k in per_kernel},
                     "iteration_frac": round(it_frac, 4),
                     "iteration_bytes_per_voxel": BYTES_PER_VOXEL_ITER},
        "e2e": {"value": round(e2e_val, 4), "unit": "Gvoxel/s",
                "h2d_bytes_per_step": 2 * pairs * nvox * 4,
                "d2h_bytes_per_step": 3 * pairs * nvox * 4,
                "iters_per_step": e2e_iters, "steps": pipe_steps,
                "path": "wlm_engine_load(host) + wlm_engine_iterate + wlm_engine_get_warp(host)",
                "overlap": "two engines alternate steps: step k+1's input copy and step k's warp "
                           "copy overlap the other engine's iterations",
                "serial_value": round(serial_val, 4),
                "serial": "one engine, one step after the other (copies not overlapped)"},
        "gpu_launches": int(launches_timed),
        "clocks": clk.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if extra:
        line["pyramid_configs"] = extra
    if rank == 0 and world == 1 and args.table6:
        line["table6"] = table6(ctx)
    traffic = load_traffic(dom)
    if traffic:
        line["roofline"]["traffic"] = traffic
    eng.close()
    return line


def run_slabs(args, rank, world, local):
    """Config 5: one large volume (default 1024^3) split into `world` z-slabs,
    one per GPU (NCCL halo exchange + plane-sum/max all-reduce); at N=1 the
    same group with one slab.  Strong scaling (the volume is fixed)."""
    import ctypes as C

    import torch

    import paper_2603_19371_b200 as P
    from paper_2603_19371_b200 import slabs
    from paper_2603_19371_b200._lib import Dims, SynthSpec

    torch.cuda.set_device(local)
    n = args.size
    shape = (n, n, n)
    nvox = n ** 3
    ctx = P.Context(local)
    lib = P.load()
    cfg = P.reg_config(nlevels=1, factors=[1], iters=[args.steps])
    # identical synthetic pair on every rank (seed 7, warp_max 16 at 1024^3,
    # SURVEY 8(d); scaled with the size below 512^3, where 16 voxels fold)
    F_d = torch.empty(shape, dtype=torch.float32, device=f"cuda:{local}")
    M_d = torch.empty(shape, dtype=torch.float32, device=f"cuda:{local}")
    spec = SynthSpec(Dims(n, n, n), 96, 0.0, 16.0 if n >= 512 else 16.0 * n / 1024, 0.01, 7)
    ctx.check(lib.wlm_synth_pair(ctx.h, C.byref(spec), F_d.data_ptr(), M_d.data_ptr(), None, 1))
    if world > 1:
        import torch.distributed as dist
        uid = slabs.broadcast_unique_id(slabs.nccl_unique_id)
        grp = slabs.RankSlab(shape, rank, world, uid, cfg=cfg, ctx=ctx)
    else:
        grp = P.SlabGroup(shape, 1, cfg=cfg, ctx=ctx)
    grp_fused = grp.fused_halos()
    grp.load(F_d, M_d)
    F_h = F_d.cpu().pin_memory() if args.e2e_iters > 0 else None
    M_h = M_d.cpu().pin_memory() if args.e2e_iters > 0 else None
    del F_d, M_d
    torch.cuda.empty_cache()
    stream = torch.cuda.ExternalStream(ctx.stream(), device=f"cuda:{local}")
    grp.set_warp(None)
    grp.begin_level(0)
    grp.iterate(args.warmup)
    ctx.synchronize()

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(world, local)
    torch.cuda.synchronize()
    launches_before = ctx.launches
    with ClockSampler(local) as clk:
        ev0.record(stream)
        grp.iterate(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(world, local)
    launches_timed = ctx.launches - launches_before
    ms_max = max_over_ranks(ev0.elapsed_time(ev1), world, local)
    st = grp.state()
    assert math.isfinite(st["r"]), st

    e2e = None
    if args.e2e_iters > 0:
        U_h = torch.empty((3,) + shape, dtype=torch.float32, pin_memory=True)
        barrier(world, local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        grp.load(F_h, M_h)
        grp.set_warp(None)
        grp.reset()  # a fresh registration: lambda0, empty loss history
        grp.begin_level(0)
        grp.iterate(args.e2e_iters)
        grp.get_warp(U_h)
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, local)
        e2e = {"value": round(nvox * args.e2e_iters / e2e_s / 1e9, 4), "unit": "Gvoxel/s",
               "h2d_bytes_per_step": 2 * nvox * 4, "d2h_bytes_per_step": 3 * nvox * 4 // world,
               "iters_per_step": args.e2e_iters,
               "path": "wlm_slab_group_load(host) + begin_level + iterate + get_warp(host, owned planes)"}

    hbm, peak_kind = peaks()
    value = nvox * args.steps / (ms_max * 1e-3) / 1e9
    it_frac = BYTES_PER_VOXEL_ITER * value / hbm / max(world, 1)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gvoxel/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "storage_dtype": "f32",
        "data": f"synthetic (GPU synth_pair, 96 blobs, smoothed random warp, max {spec.warp_max:g} voxels, seed 7)",
        "config": {"workload": f"config 5: one {n}^3 pair, z-slab sharded over {world} GPU(s), LNCC r=2 + "
                               f"pointwise LM, rejection off",
                   "volume": list(shape), "parallelism": f"z-slab x{world} (halo exchange + NCCL all-reduce)"
                   if world > 1 else "single slab", "l2": "inputs > L2",
                   # exchanges fused into the producing kernels (bit 0 g, 1 dU_s, 2 warp, 3 A/B/E:
                   # peer-memory stores + an ordering token; include/wlm.h)
                   "fused_halos": f"{grp_fused:04b}"},
        "iters_per_s": round(args.steps / (ms_max * 1e-3), 3),
        "roofline": {"bound": "hbm", "kernel": "iteration (K1..K4 + exchanges)",
                     "achieved": round(value * BYTES_PER_VOXEL_ITER / max(world, 1), 1), "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(it_frac, 4), "traffic": None,
                     "iteration_bytes_per_voxel": BYTES_PER_VOXEL_ITER},
        "gpu_launches": int(launches_timed),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    grp.close()
    return line


def pyramid_configs(ctx, lib):
    """BASELINE configs 2 and 3 through the whole-pyramid API (wlm_register):
    config 2 (brain-shaped, [4,2,1] x [100,75,50], LNCC + LM + rejection) and
    config 3 (lung-shaped, [8,4,2,1] x [100,100,75,50]) run with LM and with
    Adam, reporting wall time (host buffers in and out) and the arena
    high-water mark -- the north star's "peak device memory next to an
    Adam-state baseline"."""
    import ctypes as C

    import numpy as np

    import paper_2603_19371_b200 as P
    from paper_2603_19371_b200._lib import Dims, SynthSpec

    def synth(nx, ny, nz, seed, wmax):
        F = np.empty((nz, ny, nx), np.float32)
        M = np.empty((nz, ny, nx), np.float32)
        spec = SynthSpec(Dims(nx, ny, nz), 12, 0.0, wmax, 0.01, seed)
        ctx.check(lib.wlm_synth_pair(ctx.h, C.byref(spec), F.ctypes.data, M.ctypes.data, None, 0))
        return F, M

    def run(F, M, cfg):
        P.register(F, M, cfg, ctx=ctx)  # warm (module load, first allocations)
        t0 = time.perf_counter()
        res = P.register(F, M, cfg, ctx=ctx)
        dt = time.perf_counter() - t0
        attempts = sum(1 + t.retries for t in res.loss_trace)
        return res, dt, attempts

    out = {}
    F, M = synth(160, 192, 224, 1, 6.0)
    cfg = P.reg_config(nlevels=3, factors=[4, 2, 1], iters=[100, 75, 50], **{"lm.rejection": 1})
    res, dt, att = run(F, M, cfg)
    out["config2"] = {"dims": [160, 192, 224], "schedule": "[4,2,1] x [100,75,50]", "rejection": True,
                      "wall_s": round(dt, 4), "attempts": att, "accepted_iters": len(res.loss_trace),
                      "attempts_per_s": round(att / dt, 1), "accepted_iters_per_s": round(len(res.loss_trace) / dt, 1),
                      "final_r": res.loss_trace[-1].r, "peak_device_bytes": res.peak_device_bytes}
    F, M = synth(224, 192, 224, 2, 8.0)
    kw = dict(nlevels=4, factors=[8, 4, 2, 1], iters=[100, 100, 75, 50])
    lm, dt_lm, _ = run(F, M, P.reg_config(**kw))
    ad, dt_ad, _ = run(F, M, P.reg_config(optimizer=P.OPT_ADAM, **kw))
    # the low-memory layout (no grad M buffer, K2 re-gathers; identical results)
    lm_l, dt_lm_l, _ = run(F, M, P.reg_config(low_memory=1, **kw))
    ad_l, dt_ad_l, _ = run(F, M, P.reg_config(optimizer=P.OPT_ADAM, low_memory=1, **kw))
    out["config3"] = {"dims": [224, 192, 224], "schedule": "[8,4,2,1] x [100,100,75,50]",
                      "lm": {"wall_s": round(dt_lm, 4), "peak_device_bytes": lm.peak_device_bytes,
                             "final_r": lm.loss_trace[-1].r},
                      "adam": {"wall_s": round(dt_ad, 4), "peak_device_bytes": ad.peak_device_bytes,
                               "final_r": ad.loss_trace[-1].r},
                      "lm_memory_saving": round(1 - lm.peak_device_bytes / ad.peak_device_bytes, 4),
                      "low_memory_layout": {
                          "lm": {"wall_s": round(dt_lm_l, 4), "peak_device_bytes": lm_l.peak_device_bytes,
                                 "final_r": lm_l.loss_trace[-1].r},
                          "adam": {"wall_s": round(dt_ad_l, 4), "peak_device_bytes": ad_l.peak_device_bytes,
                                   "final_r": ad_l.loss_trace[-1].r},
                          "lm_memory_saving": round(1 - lm_l.peak_device_bytes / ad_l.peak_device_bytes, 4),
                          "note": "wlm_reg_config.low_memory = 1: K2 re-gathers grad M(x+u) instead of "
                                  "reading K1a's fp64 copy (24 B/voxel less); bit-identical results"},
                      "state_bytes": {"lm": P.state_bytes(P.OPT_LM, (224, 192, 224)),
                                      "adam": P.state_bytes(P.OPT_ADAM, (224, 192, 224))}}
    return out


def table6(ctx, sizes=(64, 128, 192, 256, 320, 384, 448, 512), steps=20):
    """PAPER.md:585-610 (Table 6, FireANTs on an A6000: Adam vs LM peak memory
    and time per step on N^3) on this engine: one pair per size, peak device
    memory of the engine (arena high-water mark) and CUDA-event time per LM
    attempt, for LM and Adam, in the default and the low-memory layouts."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2603_19371_b200 as P
    from paper_2603_19371_b200._lib import Dims, SynthSpec
    lib = P.load()
    rows = []
    for n in sizes:
        F = np.empty((n, n, n), np.float32)
        M = np.empty((n, n, n), np.float32)
        spec = SynthSpec(Dims(n, n, n), 12, 0.0, min(6.0, n / 32.0), 0.01, 5)
        ctx.check(lib.wlm_synth_pair(ctx.h, C.byref(spec), F.ctypes.data, M.ctypes.data, None, 0))
        row = {"n": n}
        for lean in (0, 1):
            for name, opt in (("lm", P.OPT_LM), ("adam", P.OPT_ADAM)):
                c = P.Context(0)
                cfg = P.reg_config(nlevels=1, factors=[1], iters=[steps + 3], optimizer=opt, low_memory=lean)
                eng = P.Engine((n, n, n), pairs=1, cfg=cfg, ctx=c)
                eng.load(F[None], M[None])
                eng.set_warp(None)
                eng.begin_level(0)
                eng.iterate(3)
                c.synchronize()
                stream = torch.cuda.ExternalStream(c.stream(), device="cuda:0")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                eng.iterate(steps)
                e1.record(stream)
                e1.synchronize()
                key = name + ("_lowmem" if lean else "")
                row[key + "_peak_bytes"] = c.peak_bytes
                row[key + "_ms_per_step"] = round(e0.elapsed_time(e1) / steps, 4)
                eng.close()
                c.close()
        for sfx in ("", "_lowmem"):
            row["lm_saving" + sfx] = round(1 - row["lm" + sfx + "_peak_bytes"] / row["adam" + sfx + "_peak_bytes"], 4)
            row["adam_over_lm_time" + sfx] = round(row["adam" + sfx + "_ms_per_step"] /
                                                   row["lm" + sfx + "_ms_per_step"], 3)
        rows.append(row)
    return rows


def load_traffic(kernel):
    """DRAM bytes per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(kernel)
        except Exception:
            return None
    return None


def host_cpu():
    """nproc and the CPU model of the box (SURVEY §8(d) CPU-baseline note)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


def _cpu_kind():
    import oracle as O
    return "reference" if O.have_ref() else "port"


def cpu_registrations(data, iters):
    """One single-threaded registration per (F, M) pair, all pairs in parallel
    (one per host core): each runs its level's initial residual, then `iters`
    LM attempts.  The reference code is serial, so the host cores are used by
    running independent registrations side by side.
    Returns the per-pair arrays of attempt wall times (initial residual
    excluded: a steady-state iteration evaluates one residual)."""
    import numpy as np

    import oracle as O
    kind = _cpu_kind()
    L = O.lib(kind)
    L.orc_set_threads(1)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[iters])
    out = [None] * len(data)

    def one(i):
        F, M = data[i]
        F = np.ascontiguousarray(F, np.float64)
        M = np.ascontiguousarray(M, np.float64)
        rc, _, _, ts = O.lm_run_level_timed(F, M, np.zeros(F.shape + (3,)), cfg, iters, kind=kind)
        out[i] = ts

    th = [threading.Thread(target=one, args=(i,)) for i in range(len(data))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    L.orc_set_threads(min(8, os.cpu_count() or 1))
    return out, kind


def cpu_baseline_sample(pairs_data, warm=2, timed=5):
    """Reference CPU path (oracle/_ref: the reference's own field.cpp
    primitives + the restated LNCC/LM modules) on the box's host cores, on
    the same workload's first pairs (the GPU-generated inputs): one
    single-threaded registration per core, each 2 warm-up + 5 timed LM
    attempts; per-iteration time = the median of the 5, step
    time = the slowest core's."""
    import numpy as np
    cores = os.cpu_count() or 1
    data = pairs_data[:min(cores, len(pairs_data))]
    t0 = time.perf_counter()
    times, kind = cpu_registrations(data, warm + timed)
    wall = time.perf_counter() - t0
    per_pair = [float(np.median(t[warm:warm + timed])) for t in times]
    step_s = max(per_pair)
    nvox = data[0][0].size
    value = len(data) * nvox / step_s / 1e9
    return {"value": round(value, 6), "unit": "Gvoxel/s", "cores": len(data), "kind": kind,
            "sample": f"{len(data)} pairs of the workload ({data[0][0].shape[0]}^3), one single-threaded "
                      f"registration per core in parallel; per pair {warm} warm-up + {timed} timed LM "
                      f"attempts after the initial residual, median attempt (SPEC.md:467); "
                      f"{wall:.0f} s wall",
            "s_per_iteration_single_thread": round(float(np.median(per_pair)), 3),
            "host": host_cpu()}


def cpu_tables():
    """SURVEY 8(d) CPU tables on the box's host: the full config-1 oracle run
    (64^3 x 100 iterations, single thread) and the reference primitives at
    192^3 (single thread, the reference's own field.cpp functions)."""
    import ctypes as C

    import numpy as np

    import oracle as O
    out = {}
    kind = _cpu_kind()
    L = O.lib(kind)
    L.orc_set_threads(1)
    F, M, _ = O.synth_pair((64, 64, 64), 0, num_blobs=12, warp_max=3.0)
    cfg = O.default_config(nlevels=1, factors=[1], iters=[100])
    t0 = time.perf_counter()
    rc, _, tr, ts = O.lm_run_level_timed(F, M, np.zeros(F.shape + (3,)), cfg, 100, kind=kind)
    out["config1_64cubed_100_iters"] = {"wall_s": round(time.perf_counter() - t0, 3), "threads": 1,
                                        "median_iter_s": round(float(np.median(ts)), 5),
                                        "final_r": tr[-1].r, "kind": kind}
    # one 192^3 registration on all host cores: the oracle port's plane-
    # parallel loops (deterministic reductions), 2 warm-up + 5
    # timed attempts, median (SURVEY 8(d) CPU baseline 3)
    cores = os.cpu_count() or 1
    Lp = O.lib("port")
    Lp.orc_set_threads(cores)
    F2, M2, _ = O.synth_pair((192, 192, 192), 1000, num_blobs=12, warp_max=6.0)
    cfg7 = O.default_config(nlevels=1, factors=[1], iters=[7])
    rc, _, _, ts = O.lm_run_level_timed(F2, M2, np.zeros(F2.shape + (3,)), cfg7, 7, kind="port")
    Lp.orc_set_threads(min(8, cores))
    out["one_192cubed_registration_all_cores"] = {"threads": cores, "kind": "port",
                                                   "median_attempt_s": round(float(np.median(ts[2:7])), 4),
                                                   "gvoxel_per_s": round(192 ** 3 / float(np.median(ts[2:7])) / 1e9, 6)}
    if O.have_ref():
        R = O.ref_lib()
        n = 192
        rng = np.random.default_rng(0)
        vol = rng.random((n, n, n))
        u = np.ascontiguousarray(rng.normal(size=(n, n, n, 3)) * 2.0)
        v = np.ascontiguousarray(rng.normal(size=(n, n, n, 3)) * 0.3)
        Mw = np.empty((n, n, n))
        gM = np.empty((n, n, n, 3))
        out_f = np.empty_like(u)
        P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        rows = {}

        def tm(name, fn):
            t = time.perf_counter()
            fn()
            rows[name] = round(time.perf_counter() - t, 4)

        tm("warp+grad", lambda: R.ref_warp_volume(P(vol), P(u), n, n, n, P(Mw), P(gM)))
        tm("normalize (max)", lambda: R.ref_normalize_step(P(v), n, n, n, 0.4, 1e-12))
        tm("compose_warp", lambda: R.ref_compose_warp(P(u), n, n, n, P(v), n, n, n, 0.2, P(out_f)))
        tm("smooth 3ch sigma=1", lambda: R.ref_gaussian_smooth(P(u), n, n, n, 3, 1.0))
        tm("smooth 3ch sigma=0.5", lambda: R.ref_gaussian_smooth(P(u), n, n, n, 3, 0.5))
        tm("smooth 1ch sigma=1", lambda: R.ref_gaussian_smooth(P(vol), n, n, n, 1, 1.0))
        tm("jacobian_det_min", lambda: R.ref_jacobian_det_min(P(u), n, n, n))
        rows["sum"] = round(sum(rows.values()), 4)
        out["reference_primitives_192_s"] = rows
    L.orc_set_threads(min(8, os.cpu_count() or 1))
    out["host"] = host_cpu()
    return out


# ------------------------------------------------------------- reference ----
def run_reference(args, rank, world):
    """The reference CPU implementation on the box's host cores: reference
    field.cpp primitives (oracle/_ref) + the restated spec-only modules, one
    single-threaded registration per core, pairs in parallel.  A step is one
    LM attempt of every sampled pair (the slowest core's attempt time); the
    levels' initial residuals are excluded, as in the GPU arm, whose timed
    steps are attempts only."""
    import numpy as np

    import oracle as O
    n = args.size
    shape = (n, n, n)
    nvox = n ** 3
    cores = os.cpu_count() or 1
    gb = args.global_batch if not args.pairs_per_gpu else args.pairs_per_gpu * world
    npairs = min(gb, cores)
    t0 = time.perf_counter()
    data = [O.synth_pair(shape, 1000 + p, num_blobs=12, warp_max=warp_max(n))[:2] for p in range(npairs)]
    t_synth = time.perf_counter() - t0
    # bound the sample: as many steps as fit the budget at the measured rate
    # (one probe attempt per pair first)
    warm = max(1, min(args.warmup, 2))
    probe, kind = cpu_registrations(data, 1)
    per_attempt = max(max(t) for t in probe)
    steps = max(1, min(args.steps, int(args.ref_budget_s / max(per_attempt, 1e-9)) - warm))
    times, kind = cpu_registrations(data, warm + steps)
    step_s = [max(t[k] for t in times) for k in range(warm, warm + steps)]
    dt = float(sum(step_s))
    value = npairs * nvox * steps / dt / 1e9
    sample = (f"{steps} steps x 1 LM attempt of {npairs} pairs of {n}^3 (oracle synth_pair seeds 1000+), "
              f"one single-threaded registration per host core; step = the slowest pair's attempt; "
              f"{warm} warm-up attempts and the initial residual excluded; inputs made in {t_synth:.0f} s")
    return {
        "metric": METRIC, "value": round(value, 6), "unit": "Gvoxel/s", "n_gpus": world,
        "steps": args.steps, "steps_timed": steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3 / steps, 1), "higher_is_better": True,
        "scaling": "strong" if not args.pairs_per_gpu else "weak", "vs_baseline": None,
        "dtype": "f64", "impl": "reference",
        "data": "synthetic (oracle synth_pair: Gaussian blobs + smoothed random warp max 6, noise 0.01, "
                "seeds 1000+)",
        "config": config4(n, gb, world),
        "cpu_baseline": {"value": round(value, 6), "unit": "Gvoxel/s", "cores": npairs, "kind": kind,
                         "sample": sample, "s_per_iteration_single_thread":
                             round(float(np.median(step_s)), 3), "host": host_cpu()},
        "e2e": {"value": round(value, 6), "unit": "Gvoxel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=192)
    ap.add_argument("--global-batch", type=int, default=64, help="config 4: pairs split over the GPUs")
    ap.add_argument("--pairs-per-gpu", type=int, default=0,
                    help="fixed pairs per GPU instead (weak scaling); 0 = global batch / N")
    ap.add_argument("--low-memory", type=int, default=0,
                    help="wlm_reg_config.low_memory: 1 = no grad M buffer, K2 re-gathers (identical results)")
    ap.add_argument("--table6", action="store_true",
                    help="add PAPER.md Table 6's memory / time comparison (LM vs Adam, 64^3 .. 512^3)")
    ap.add_argument("--cpu-tables", action="store_true",
                    help="add the config-1 run and the 192^3 primitive table to cpu_baseline")
    ap.add_argument("--e2e-iters", type=int, default=100)
    ap.add_argument("--e2e-groups", type=int, default=2, help="pair groups of each pipelined e2e engine")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 2/3 pyramid runs")
    ap.add_argument("--ref-budget-s", type=float, default=200.0)
    ap.add_argument("--config", type=int, default=4, choices=[4, 5],
                    help="4: batch of 192^3 pairs (default, weak scaling); 5: one 1024^3 volume in z-slabs")
    args = ap.parse_args()
    if args.config == 5 and args.size == 192:
        args.size = 1024
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", 0))
        world = int(os.environ.get("WORLD_SIZE", 1))
        if rank != 0:
            return
        print(json.dumps(run_reference(args, rank, world)), flush=True)
        return

    rank, world, local = dist_init(args.gpus)
    line = (run_slabs if args.config == 5 else run_ours)(args, rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
