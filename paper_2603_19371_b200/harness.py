"""The reference's harness module over the GPU path:
``synth``, ``register``, ``sweep``, ``membench`` and ``reject-ablation``,
each a function here and a subcommand of ``python -m paper_2603_19371_b200``.

Every registration, synthetic pair and endpoint-error warp inversion runs on
the device through the public API (warplm.py / engine.py).  The host only
parses configs, reduces endpoint errors and writes the versioned CSV
(``# warplm-csv v1``).

Ground truth for endpoint errors: ``synth_pair``'s moving image is the fixed
image sampled through Id + u_true and ``register`` solves
M o (Id + u) ~ F, so the warp to compare with is the inverse displacement
u_gt (u_gt(x) = -u_true(x + u_gt(x))), computed on the device by fixed-point
iteration of compose_warp.
"""
from __future__ import annotations

import csv
import math
import os
import statistics
import sys
import time

import numpy as np

from ._lib import DimensionMismatch, InvalidArgument
from .io import IoError, read_dsp3, read_vol3, write_dsp3, write_vol3, write_trace_csv
from .warplm import (Context, compose_warp, default_context, reg_config, register, state_bytes,
                     synth_pair)

CSV_HEADER = "# warplm-csv v1"

__all__ = ["ConfigError", "parse_config", "load_config", "endpoint_error", "inverse_displacement",
           "cmd_synth", "cmd_register", "cmd_sweep", "cmd_membench", "cmd_reject_ablation",
           "SWEEP_COLUMNS", "MEMBENCH_COLUMNS", "ABLATION_COLUMNS"]


class ConfigError(ValueError):
    """Malformed key=value config (exit code 2)."""


# --------------------------------------------------------------- config ----
_LM = ("lambda0", "mu_plus", "mu_minus", "tile_size", "rejection", "tau", "lambda_max", "max_retries")
_ADAM = ("beta1", "beta2", "eps_hat", "lr")
_TOP = ("lncc_radius", "optimizer", "gd_lr", "nlevels", "factors", "iters", "target_max_disp",
        "step_floor", "sigma_update", "sigma_warp", "log_jacobian", "metric", "demons_alpha",
        "mi_bins", "mi_sigma")
_ALIASES = {"rejection_enabled": "lm.rejection", "schedule": "factors"}
_ENUMS = {"optimizer": {"lm": 0, "adam": 1, "gd": 2, "demons": 3},
          "metric": {"lncc": 0, "mse": 1, "mi": 2}}
_INTS = {"tile_size", "rejection", "max_retries", "lncc_radius", "optimizer", "nlevels",
         "log_jacobian", "metric", "mi_bins"}


def _key(k):
    k = _ALIASES.get(k, k)
    if "." in k:
        grp, name = k.split(".", 1)
        if (grp == "lm" and name in _LM) or (grp == "adam" and name in _ADAM):
            return k, name
        raise ConfigError(f"unknown config key '{k}'")
    if k in _LM:
        return "lm." + k, k
    if k in _ADAM:
        return "adam." + k, k
    if k in _TOP:
        return k, k
    raise ConfigError(f"unknown config key '{k}'")


def _value(name, text):
    t = text.strip()
    if name in _ENUMS and t.lower() in _ENUMS[name]:
        return _ENUMS[name][t.lower()]
    if name in ("factors", "iters"):
        try:
            return [int(x) for x in t.replace(",", " ").split()]
        except ValueError:
            raise ConfigError(f"{name}: expected a list of integers, got '{t}'") from None
    if name in ("rejection",) and t.lower() in ("true", "false", "on", "off"):
        return int(t.lower() in ("true", "on"))
    try:
        v = float(t)
    except ValueError:
        raise ConfigError(f"{name}: expected a number, got '{t}'") from None
    if name in _INTS:
        if v != int(v):
            raise ConfigError(f"{name}: expected an integer, got '{t}'")
        return int(v)
    return v


def parse_config(text: str) -> dict:
    """Plain ``key = value`` lines: every LmConfig / RegConfig
    field addressable, ``lm.`` / ``adam.`` prefixes optional, ``#`` comments,
    lists comma- or space-separated, optimizer / metric by name or number.
    Returns keyword arguments for ``reg_config``."""
    kw = {}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {ln}: expected key=value, got '{raw.strip()}'")
        k, v = (s.strip() for s in line.split("=", 1))
        full, name = _key(k)
        kw[full] = _value(name, v)
    if "factors" in kw and "nlevels" not in kw:
        kw["nlevels"] = len(kw["factors"])
    return kw


def load_config(path: str | None, **overrides) -> dict:
    kw = {}
    if path:
        try:
            with open(path) as f:
                kw = parse_config(f.read())
        except OSError as e:
            raise ConfigError(f"{path}: {e.strerror}") from None
    kw.update(overrides)
    return kw


def _reg_config(kw):
    try:
        return reg_config(**kw)
    except (TypeError, AttributeError, IndexError) as e:
        raise ConfigError(str(e)) from None


# ------------------------------------------------------- endpoint error ----
def inverse_displacement(u_true, iters=300, tol=1e-6, ctx=None):
    """u_gt = (Id + u_true)^-1 - Id on the device: w <- w - compose(u_true, w, 1)
    (= -u_true(x + w)); converges away from the clamped border, which the
    endpoint error excludes."""
    u = np.asarray(u_true, np.float64)
    w = -u.copy()
    for _ in range(iters):
        res = compose_warp(u, w, 1.0, ctx=ctx)  # w + u(x + w)
        w = w - res
        if np.abs(res[2:-2, 2:-2, 2:-2]).max(initial=0.0) < tol:
            break
    return w


def endpoint_error(u_est, u_true):
    """(mean, max) per-voxel Euclidean distance over the centre, 2-voxel
    border excluded."""
    a, b = np.asarray(u_est, np.float64), np.asarray(u_true, np.float64)
    if a.shape != b.shape:
        raise DimensionMismatch(2, "endpoint_error: dimension mismatch")
    d = np.linalg.norm(a - b, axis=-1)[2:-2, 2:-2, 2:-2]
    if d.size == 0:
        return float("nan"), float("nan")
    return float(d.mean()), float(d.max())


# -------------------------------------------------------------- commands ----
def cmd_synth(dims, seed, out_dir, num_blobs=12, warp_max=3.0, warp_sigma=0.0, noise_sigma=0.01,
              ctx=None):
    """synth_pair -> fixed.vol3, moving.vol3, u_true.dsp3 in out_dir."""
    nx, ny, nz = dims
    if warp_max < 0 or num_blobs < 0 or noise_sigma < 0 or warp_sigma < 0:
        raise ConfigError("synth: parameters must be >= 0")
    if warp_max >= min(dims) / 4:
        raise ConfigError(f"synth: warp_max {warp_max} must be < min(dims)/4 (SPEC.md:408)")
    F, M, U = synth_pair((nz, ny, nx), seed, num_blobs, warp_max, noise_sigma, warp_sigma, ctx=ctx)
    os.makedirs(out_dir, exist_ok=True)
    paths = {k: os.path.join(out_dir, f) for k, f in
             (("fixed", "fixed.vol3"), ("moving", "moving.vol3"), ("u_true", "u_true.dsp3"))}
    write_vol3(paths["fixed"], F)
    write_vol3(paths["moving"], M)
    write_dsp3(paths["u_true"], np.ascontiguousarray(np.moveaxis(U, -1, 0)))
    return paths


def cmd_register(fixed_path, moving_path, out_dir, cfg_kw=None, csv_path=None, truth_path=None,
                 ctx=None):
    """cmd_register: VOL3 pair in; warp.dsp3 and the CSV
    trace out; returns the summary (also the stdout line of the CLI).  With
    ``truth_path`` (a synth u_true.dsp3) the summary has the endpoint error."""
    F = read_vol3(fixed_path)
    M = read_vol3(moving_path)
    if F.shape != M.shape:
        raise DimensionMismatch(2, f"{fixed_path}, {moving_path}: dimension mismatch")
    cfg = _reg_config(cfg_kw or {})
    res = register(F, M, cfg, ctx=ctx)
    os.makedirs(out_dir, exist_ok=True)
    warp_path = os.path.join(out_dir, "warp.dsp3")
    write_dsp3(warp_path, np.ascontiguousarray(np.moveaxis(res.final_warp, -1, 0), dtype=np.float32))
    csv_path = csv_path or os.path.join(out_dir, "trace.csv")
    write_trace_csv(csv_path, res.loss_trace)
    last = res.loss_trace[-1] if res.loss_trace else None
    summary = dict(warp=warp_path, csv=csv_path, steps=len(res.loss_trace),
                   final_r=last.r if last else float("nan"),
                   final_loss_raw=last.loss_raw if last else float("nan"),
                   final_lambda=last.lam if last else float("nan"),
                   retries=sum(t.retries for t in res.loss_trace),
                   jac_det_min=res.jac_det_min_final,
                   max_disp=float(np.abs(res.final_warp).max()) if res.final_warp.size else 0.0)
    if truth_path:
        U = np.moveaxis(read_dsp3(truth_path), 0, -1)
        if U.shape[:3] != F.shape:
            raise DimensionMismatch(2, f"{truth_path}: dimension mismatch")
        summary["mean_epe"], summary["max_epe"] = endpoint_error(
            res.final_warp, inverse_displacement(U, ctx=ctx))
    return summary


def _write_csv(path, columns, rows):
    with open(path, "w", newline="", encoding="utf-8") as f:
        f.write(CSV_HEADER + "\n")
        w = csv.writer(f)
        w.writerow(columns)
        for r in rows:
            w.writerow([_fmt(r.get(c, "")) for c in columns])


def _fmt(v):
    if isinstance(v, float):
        return repr(v) if math.isfinite(v) else ("inf" if v > 0 else "-inf" if v < 0 else "nan")
    return v


def _suite_pair(dims, seed, warp_max, ctx, cache):
    """Synthetic pair + inverse ground truth, generated once per sweep."""
    key = (tuple(dims), seed, warp_max)
    if key not in cache:
        nx, ny, nz = dims
        F, M, U = synth_pair((nz, ny, nx), seed, 12, warp_max, 0.01, 0.0, ctx=ctx)
        cache[key] = (F, M, inverse_displacement(U, ctx=ctx))
    return cache[key]


SWEEP_COLUMNS = ("param", "value", "repeat", "final_loss", "mean_epe", "max_epe", "final_lambda",
                 "steps_rejected")
_SWEEP_PARAMS = {"lambda0": "lm.lambda0", "mu_plus": "lm.mu_plus", "mu_minus": "lm.mu_minus",
                 "tile_size": "lm.tile_size"}


def cmd_sweep(param, values, repeats=1, cfg_kw=None, dims=(32, 32, 32), seed=0, warp_max=3.0,
              csv_path=None, ctx=None):
    """cmd_sweep: one registration per value x repeat on the
    fixed synthetic pairs (repeat i uses seed + i).  A failing run writes a
    NaN row and the sweep continues.  Rows in spec order."""
    if param not in _SWEEP_PARAMS:
        raise ConfigError(f"sweep: parameter must be one of {sorted(_SWEEP_PARAMS)}")
    if not values:
        raise ConfigError("sweep: empty value list")
    ctx = ctx or default_context()
    rows, pairs = [], {}
    for v in values:
        for rep in range(repeats):
            row = dict(param=param, value=v, repeat=rep)
            try:
                F, M, ugt = _suite_pair(dims, seed + rep, warp_max, ctx, pairs)
                kw = dict(cfg_kw or {})
                kw[_SWEEP_PARAMS[param]] = int(v) if param == "tile_size" else float(v)
                res = register(F, M, _reg_config(kw), ctx=ctx)
                mean, mx = endpoint_error(res.final_warp, ugt)
                row.update(final_loss=res.loss_trace[-1].r, mean_epe=mean, max_epe=mx,
                           final_lambda=res.loss_trace[-1].lam,
                           steps_rejected=sum(t.retries for t in res.loss_trace))
            except (InvalidArgument, ConfigError, RuntimeError) as e:
                print(f"sweep {param}={v} repeat {rep}: {e}", file=sys.stderr)
                row.update(final_loss=float("nan"), mean_epe=float("nan"), max_epe=float("nan"),
                           final_lambda=float("nan"), steps_rejected=-1)
            rows.append(row)
    if csv_path:
        _write_csv(csv_path, SWEEP_COLUMNS, rows)
    return rows


MEMBENCH_COLUMNS = ("n", "state_bytes_lm", "state_bytes_adam", "ms_per_step_lm", "ms_per_step_adam",
                    "note")


def _step_ms(F, M, opt, warm=2, timed=5):
    from .engine import Engine
    c = Context(0)
    try:
        e = Engine(F.shape, 1, reg_config(optimizer=opt), ctx=c)
        try:
            e.load(F[None], M[None])
            e.set_warp(None)
            e.begin_level(0)
            for _ in range(warm):
                e.step()
            c.synchronize()
            ts = []
            for _ in range(timed):
                t0 = time.perf_counter()
                e.step()
                c.synchronize()
                ts.append((time.perf_counter() - t0) * 1e3)
            return statistics.median(ts)  # median of 5 after 2 warm-up
        finally:
            e.close()
    finally:
        c.close()


def cmd_membench(sizes, csv_path=None, ctx=None):
    """cmd_membench: per N, optimizer-state bytes (fp32
    elements) and the median wall time of one LM / Adam step on an N^3 pair."""
    rows = []
    for n in sizes:
        row = dict(n=n, state_bytes_lm=state_bytes(0, (n, n, n)), state_bytes_adam=state_bytes(1, (n, n, n)),
                   note="")
        try:
            F, M, _ = synth_pair((n, n, n), 7, 12, min(3.0, n / 4 - 0.5), 0.01, 0.0, ctx=ctx)
            row["ms_per_step_lm"] = _step_ms(F, M, 0)
            row["ms_per_step_adam"] = _step_ms(F, M, 1)
        except (InvalidArgument, RuntimeError) as e:  # allocation failure etc.: skip with a note
            row.update(ms_per_step_lm=float("nan"), ms_per_step_adam=float("nan"), note=str(e))
        rows.append(row)
    if csv_path:
        _write_csv(csv_path, MEMBENCH_COLUMNS, rows)
    return rows


ABLATION_COLUMNS = ("pair", "warp_max", "variant", "final_loss", "final_lambda", "max_lambda", "retries",
                    "floor_steps", "lambda_trace")
_VARIANTS = (("no-rejection", {"lm.rejection": 0}),
             ("rejection+cap=1.0", {"lm.rejection": 1, "lm.lambda_max": 1.0}),
             ("rejection+cap=inf", {"lm.rejection": 1, "lm.lambda_max": float("inf")}))


def cmd_reject_ablation(cfg_kw=None, dims=(32, 32, 32), seeds=(0, 1, 2), hard_warp_max=7.0,
                        easy_warp_max=3.0, csv_path=None, ctx=None):
    """cmd_reject_ablation: {no-rejection, rejection + cap
    1.0, rejection + cap inf} on easy pairs plus one engineered hard pair
    (large warp_max).  ``floor_steps`` counts iterations whose smoothed update
    fell below the normalisation floor: its applied step is then
    0.4 max|du| / floor instead of 0.4 voxels (the runaway-lambda stall)."""
    ctx = ctx or default_context()
    nx, ny, nz = dims
    pairs = [(f"easy-{s}", s, easy_warp_max, 0.0) for s in seeds]
    pairs.append(("hard", 11, hard_warp_max, min(dims) / 8.0))
    rows = []
    for name, seed, wm, ws in pairs:
        F, M, _ = synth_pair((nz, ny, nx), seed, 12, wm, 0.01, ws, ctx=ctx)
        for variant, over in _VARIANTS:
            kw = dict(cfg_kw or {})
            kw.update(over)
            cfg = _reg_config(kw)
            res = register(F, M, cfg, ctx=ctx)
            tr = res.loss_trace
            floor_eps = cfg.target_max_disp / cfg.step_floor
            rows.append(dict(pair=name, warp_max=wm, variant=variant, final_loss=tr[-1].r,
                             final_lambda=tr[-1].lam, max_lambda=max(t.lam for t in tr),
                             retries=sum(t.retries for t in tr),
                             floor_steps=sum(1 for t in tr if t.eps >= floor_eps),
                             lambda_trace=";".join(repr(t.lam) for t in tr)))
    if csv_path:
        _write_csv(csv_path, ABLATION_COLUMNS, rows)
    return rows


# ------------------------------------------------------------------ CLI ----
def main(argv=None) -> int:
    """CLI: exit 0 success, 1 runtime failure, 2 input error."""
    import argparse
    ap = argparse.ArgumentParser(prog="python -m paper_2603_19371_b200",
                                 description="warplm harness on the B200 path (SPEC.md:399-477)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    s = sub.add_parser("synth", help="synthetic pair -> fixed.vol3, moving.vol3, u_true.dsp3")
    s.add_argument("--dims", type=int, nargs=3, default=[32, 32, 32], metavar=("NX", "NY", "NZ"))
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--num-blobs", type=int, default=12)
    s.add_argument("--warp-max", type=float, default=3.0)
    s.add_argument("--warp-sigma", type=float, default=0.0)
    s.add_argument("--noise-sigma", type=float, default=0.01)
    s.add_argument("--out-dir", required=True)

    r = sub.add_parser("register", help="register FIXED.vol3 MOVING.vol3 -> warp.dsp3 + CSV trace")
    r.add_argument("fixed")
    r.add_argument("moving")
    r.add_argument("--config")
    r.add_argument("--truth", help="u_true.dsp3 from synth: adds the endpoint error")
    r.add_argument("--out-dir", required=True)
    r.add_argument("--csv")

    w = sub.add_parser("sweep", help="hyperparameter sweep on synthetic pairs -> CSV")
    w.add_argument("--param", required=True, choices=sorted(_SWEEP_PARAMS))
    w.add_argument("--values", required=True, help="comma-separated")
    w.add_argument("--repeats", type=int, default=1)
    w.add_argument("--config")
    w.add_argument("--seed", type=int, default=0)
    w.add_argument("--dims", type=int, nargs=3, default=[32, 32, 32])
    w.add_argument("--warp-max", type=float, default=3.0)
    w.add_argument("--csv", required=True)

    m = sub.add_parser("membench", help="optimizer state bytes and step time per N^3")
    m.add_argument("--sizes", default="32,64")
    m.add_argument("--csv", required=True)

    a = sub.add_parser("reject-ablation", help="rejection / cap ablation -> CSV")
    a.add_argument("--config")
    a.add_argument("--seed", type=int, default=0)
    a.add_argument("--dims", type=int, nargs=3, default=[32, 32, 32])
    a.add_argument("--csv", required=True)

    args = ap.parse_args(argv)
    try:
        if args.cmd == "synth":
            paths = cmd_synth(args.dims, args.seed, args.out_dir, args.num_blobs, args.warp_max,
                              args.warp_sigma, args.noise_sigma)
            print(" ".join(f"{k}={v}" for k, v in paths.items()))
        elif args.cmd == "register":
            summ = cmd_register(args.fixed, args.moving, args.out_dir, load_config(args.config), args.csv,
                                args.truth)
            print(" ".join(f"{k}={_fmt(v)}" for k, v in summ.items()))
        elif args.cmd == "sweep":
            try:
                vals = [float(v) for v in args.values.split(",") if v.strip()]
            except ValueError:
                raise ConfigError(f"sweep: bad --values '{args.values}'") from None
            rows = cmd_sweep(args.param, vals, args.repeats, load_config(args.config), tuple(args.dims),
                             args.seed, args.warp_max, args.csv)
            print(f"sweep: {len(rows)} rows -> {args.csv}")
        elif args.cmd == "membench":
            try:
                sizes = [int(v) for v in args.sizes.split(",") if v.strip()]
            except ValueError:
                raise ConfigError(f"membench: bad --sizes '{args.sizes}'") from None
            rows = cmd_membench(sizes, args.csv)
            print(f"membench: {len(rows)} rows -> {args.csv}")
        else:
            rows = cmd_reject_ablation(load_config(args.config), tuple(args.dims),
                                       tuple(args.seed + i for i in range(3)), csv_path=args.csv)
            print(f"reject-ablation: {len(rows)} rows -> {args.csv}")
    except (IoError, ConfigError, DimensionMismatch, InvalidArgument) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # runtime failure (CUDA, non-finite loss, ...)
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0
