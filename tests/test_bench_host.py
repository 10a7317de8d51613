"""bench.py's multi-rank plumbing (barrier, max over ranks) and its JSON
contract on the host: world_size-2 gloo processes, no GPU."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        bench.barrier(world, 0)
        got = bench.max_over_ranks(10.0 + rank, world, 0)  # each rank's timing
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_max_over_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    got = dict(q.get(timeout=5) for _ in range(world))
    assert all(v == 10.0 + world - 1 for v in got.values())


def test_reference_arm_other_ranks_exit_silently():
    """Under torchrun only rank 0 runs and prints the reference line."""
    import subprocess
    import sys
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_reference_arm_line_and_config_match_ours():
    """The reference arm (CPU) prints the contract's line with the same
    `config` object our arm uses (bench.config4), attempts only in its
    timed steps, and a cpu_baseline describing the sample."""
    import json
    import subprocess
    import sys
    sys.path.insert(0, ROOT)
    import bench
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--size", "24", "--global-batch", "2"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "Gvoxel/s"
    assert line["config"] == bench.config4(24, 2, 1)
    assert line["steps_timed"] == 2 and line["cpu_baseline"]["cores"] == min(2, os.cpu_count())
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_cpu_registrations_time_attempts_only():
    """Attempt timings exclude the level's initial residual: k attempts give
    k timings, each positive."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import oracle as O
    F, M, _ = O.synth_pair((16, 16, 16), 3, num_blobs=4, warp_max=1.0)
    times, kind = bench.cpu_registrations([(F, M), (F, M)], 3)
    assert len(times) == 2 and all(len(t) == 3 and (t > 0).all() for t in times)
