"""A wider seeded sweep of the slab-invariance property (GPU; not part of
pytest: minutes): N random configurations of tests/test_gpu_parity.py's
fuzzer through in-process z-slab groups of 2-5 slabs, with the fused halo
stores and with the copy exchange, each bit-identical to the single-domain
engine.  Prints one line per case and a summary.

    python tools/slab_sweep.py [N] [first_seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from test_gpu_parity import _fuzz_case, run_engine, same_trace  # noqa: E402


def main():
    import paper_2603_19371_b200 as P
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    ctx = P.Context(0)
    fails, tested = [], 0
    for case in range(first, first + n):
        shape, kw, warp_max, seed = _fuzz_case(case)
        shape = (max(shape[0], 24),) + shape[1:]
        for attempt in range(6):
            try:
                F, M, _ = O.synth_pair(shape, seed, num_blobs=6, warp_max=warp_max / 2 ** attempt)
                break
            except ValueError:
                continue
        else:
            continue
        cfg = P.reg_config(**kw)
        w1, (t1,), _ = run_engine(P, ctx, F, M, cfg, 8)
        for fused in ("1", "0"):
            os.environ["WLM_SLAB_FUSED"] = fused
            for ns in (2, 3, 4, 5):
                try:
                    grp = P.SlabGroup(F.shape, ns, cfg=cfg, ctx=ctx)
                except P.InvalidArgument:
                    continue
                mask = grp.fused_halos()
                grp.load(F, M)
                grp.set_warp(None)
                grp.begin_level(0)
                grp.iterate(8)
                w, t = grp.get_warp(), grp.trace()
                grp.close()
                ok = same_trace(t, t1) and np.array_equal(w, w1[0])
                tested += 1
                if not ok:
                    fails.append((case, fused, ns, shape, kw))
                print(case, shape, fused, ns, f"mask={mask:04b}", "ok" if ok else "MISMATCH", flush=True)
    print(f"summary: {tested} slab runs, {len(fails)} mismatches", fails[:5])
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
