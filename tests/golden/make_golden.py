"""Generate tests/golden/*.npz from the UNMODIFIED reference code.

Runs in the build container only (needs oracle/_ref/liboracle_ref.so, built
from /root/reference/proj/src/{field,io}.cpp by oracle/Makefile).  The
fixtures pin the oracle's restatement of the reference `field` module
(tests/test_oracle.py checks the oracle against them bit-for-bit) and give
the GPU parity tests reference outputs that do not need /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "field_ref.npz")


def main():
    L = O.ref_lib()
    p = O._p
    rng = np.random.default_rng(20260318)
    out = {}

    # sample_trilinear_grad at random points, including knots, borders and
    # out-of-grid positions (field.cpp:43-90)
    vol = rng.normal(size=(5, 6, 7))  # (nz, ny, nx)
    pts = np.concatenate([
        rng.uniform(-2, 9, size=(200, 3)),
        rng.integers(-1, 8, size=(60, 3)).astype(np.float64),     # knots + outside
        np.array([[0, 0, 0], [6, 5, 4], [6.0, 0.5, 0.5], [3.5, 5.0, 2.0], [-1e-9, 2, 2],
                  [6 - 1e-12, 2, 2], [6 + 1e-12, 2, 2], [np.nan, 1, 1], [1, np.inf, 1]]),
    ])
    vals = np.empty(len(pts))
    grads = np.empty((len(pts), 3))
    g3 = np.empty(3)
    for i, q in enumerate(pts):
        vals[i] = L.ref_sample_trilinear_grad(p(vol), 7, 6, 5, q[0], q[1], q[2], p(g3))
        grads[i] = g3
    out.update(sample_vol=vol, sample_pts=pts, sample_val=vals, sample_grad=grads)

    # compose_warp on 6^3 / 8x7x6 random fields (field.cpp:123-142)
    for name, shape, scale, eps in [("c6", (6, 6, 6), 1.5, 0.3), ("c876", (6, 7, 8), 2.0, 0.7)]:
        u = rng.normal(size=shape + (3,)) * scale
        v = rng.normal(size=shape + (3,))
        o = np.empty_like(u)
        nz, ny, nx = shape
        assert L.ref_compose_warp(p(u), nx, ny, nz, p(v), nx, ny, nz, eps, p(o)) == 0
        out[f"{name}_u"], out[f"{name}_v"], out[f"{name}_eps"], out[f"{name}_out"] = u, v, eps, o

    # gaussian_smooth, sigma 1.0 / 0.5 / 2.3, 1 and 3 channels (field.cpp:205-269)
    for sig in (1.0, 0.5, 2.3):
        f = rng.normal(size=(9, 7, 8, 3))
        g = f.copy()
        L.ref_gaussian_smooth(p(g), 8, 7, 9, 3, sig)
        v1 = rng.normal(size=(9, 7, 8))
        w1 = v1.copy()
        L.ref_gaussian_smooth(p(w1), 8, 7, 9, 1, sig)
        key = str(sig).replace(".", "p")
        out[f"sm{key}_field_in"], out[f"sm{key}_field_out"] = f, g
        out[f"sm{key}_vol_in"], out[f"sm{key}_vol_out"] = v1, w1

    # jacobian_det_min, max_abs_component, normalize_step
    u = rng.normal(size=(7, 6, 5, 3)) * 0.2
    out["jac_u"] = u
    out["jac_out"] = L.ref_jacobian_det_min(p(u), 5, 6, 7)
    u2 = rng.normal(size=(2, 3, 2, 3)) * 0.2  # n == 2 axes (one-sided differences)
    out["jac2_u"] = u2
    out["jac2_out"] = L.ref_jacobian_det_min(p(u2), 2, 3, 2)
    out["max_out"] = L.ref_max_abs_component(p(u), 5, 6, 7)
    out["norm_out"] = L.ref_normalize_step(p(u), 5, 6, 7, 0.4, 1e-12)

    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
