"""Harness module: config files, CLI exit codes, CSV
schema (host), and the five subcommands on the GPU path."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

H = pytest.importorskip("paper_2603_19371_b200.harness")


def cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2603_19371_b200", *map(str, args)],
                          capture_output=True, text=True, cwd=cwd or ROOT, timeout=600)


def read_csv(path):
    with open(path, encoding="utf-8") as f:
        first = f.readline().rstrip("\n")
        return first, list(csv.DictReader(f))


# ----------------------------------------------------------------- host ----
def test_parse_config_every_field_addressable():
    from paper_2603_19371_b200 import reg_config
    kw = H.parse_config("""
        # comment line
        lambda0 = 0.01          # LmConfig, bare
        lm.mu_plus = 2.0        # LmConfig, prefixed
        rejection_enabled = true
        lambda_max = inf
        max_retries = 4
        tile_size = 3
        beta1 = 0.8
        adam.lr = 0.25
        optimizer = adam
        metric = mse
        factors = 4, 2, 1
        iters = 10 20 30
        sigma_update = 1.5
        sigma_warp = 0
        log_jacobian = 1
        mi_bins = 16
    """)
    c = reg_config(**kw)
    assert c.lm.lambda0 == 0.01 and c.lm.mu_plus == 2.0 and c.lm.rejection == 1
    assert c.lm.lambda_max == float("inf") and c.lm.max_retries == 4 and c.lm.tile_size == 3
    assert c.adam.beta1 == 0.8 and c.adam.lr == 0.25 and c.optimizer == 1 and c.metric == 1
    assert c.nlevels == 3 and list(c.factors)[:3] == [4, 2, 1] and list(c.iters)[:3] == [10, 20, 30]
    assert c.sigma_update == 1.5 and c.sigma_warp == 0.0 and c.log_jacobian == 1 and c.mi_bins == 16
    # untouched fields keep the SPEC defaults
    assert c.lm.mu_minus == 0.975 and c.target_max_disp == 0.4


@pytest.mark.parametrize("text", ["nonsense = 1", "lm.beta1 = 0.5", "lambda0 0.1", "tile_size = 1.5",
                                  "factors = 4, x", "lambda0 = fast"])
def test_parse_config_rejects(text):
    with pytest.raises(H.ConfigError):
        H.parse_config(text)


def test_endpoint_error_kats():
    u = np.random.default_rng(0).normal(size=(8, 8, 8, 3))
    assert H.endpoint_error(u, u) == (0.0, 0.0)
    t = np.zeros((8, 8, 8, 3)); t[..., 0] = 3.0
    assert H.endpoint_error(np.zeros_like(t), t) == (3.0, 3.0)
    # scalar-loop oracle on random fields
    a, b = u, np.random.default_rng(1).normal(size=u.shape)
    d = [np.sqrt(sum((a[z, y, x, c] - b[z, y, x, c]) ** 2 for c in range(3)))
         for z in range(2, 6) for y in range(2, 6) for x in range(2, 6)]
    m, mx = H.endpoint_error(a, b)
    assert abs(m - np.mean(d)) < 1e-12 and abs(mx - max(d)) < 1e-12


def test_cli_input_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.vol3"
    bad.write_bytes(b"XXXX" + bytes(12))
    p = cli("register", bad, bad, "--out-dir", tmp_path / "o")
    assert p.returncode == 2 and "bad magic" in p.stderr
    p = cli("register", tmp_path / "missing.vol3", bad, "--out-dir", tmp_path / "o")
    assert p.returncode == 2 and "cannot open" in p.stderr
    cfg = tmp_path / "c.cfg"
    cfg.write_text("no_such_key = 1\n")
    p = cli("register", bad, bad, "--config", cfg, "--out-dir", tmp_path / "o")
    assert p.returncode == 2 and "unknown config key" in p.stderr
    p = cli("synth", "--dims", 16, 16, 16, "--warp-max", 5, "--out-dir", tmp_path / "s")
    assert p.returncode == 2 and "warp_max" in p.stderr
    assert cli("sweep", "--param", "nope", "--values", "1", "--csv", tmp_path / "x.csv").returncode == 2
    assert cli("frobnicate").returncode == 2


def test_csv_schema_is_versioned(tmp_path):
    H._write_csv(tmp_path / "t.csv", H.SWEEP_COLUMNS,
                 [dict(param="lambda0", value=0.5, repeat=0, final_loss=float("nan"), mean_epe=1.0,
                       max_epe=2.0, final_lambda=float("inf"), steps_rejected=3)])
    first, rows = read_csv(tmp_path / "t.csv")
    assert first == "# warplm-csv v1"
    assert list(rows[0]) == list(H.SWEEP_COLUMNS)
    assert rows[0]["final_loss"] == "nan" and rows[0]["final_lambda"] == "inf"


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
def test_gpu_synth_pair_contract(ctx):
    from paper_2603_19371_b200 import jacobian_det_min, residual_mse, synth_pair
    shape = (24, 28, 32)
    a = synth_pair(shape, 5, warp_max=3.0, ctx=ctx)
    b = synth_pair(shape, 5, warp_max=3.0, ctx=ctx)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    F, M, U = a
    assert F.shape == shape and U.shape == shape + (3,)
    assert abs(np.abs(U).max() - 3.0) < 1e-5 and jacobian_det_min(U, ctx=ctx) > 0
    F0, M0, U0 = synth_pair(shape, 5, warp_max=0.0, noise_sigma=0.0, ctx=ctx)
    assert np.array_equal(F0, M0) and not U0.any()
    # noise 0: residual at the ground-truth (inverse) warp is interpolation error only
    F1, M1, U1 = synth_pair(shape, 6, warp_max=2.0, noise_sigma=0.0, ctx=ctx)
    ugt = H.inverse_displacement(U1, ctx=ctx)
    rng2 = float(F1.max() - F1.min()) ** 2
    assert residual_mse(F1, M1, ugt, gradient=False, ctx=ctx).r < 1e-3 * rng2
    assert residual_mse(F1, M1, np.zeros_like(ugt), gradient=False, ctx=ctx).r > \
        residual_mse(F1, M1, ugt, gradient=False, ctx=ctx).r


@pytest.mark.gpu
def test_cli_synth_register_roundtrip(tmp_path):
    p = cli("synth", "--dims", 32, 32, 32, "--seed", 3, "--out-dir", tmp_path)
    assert p.returncode == 0, p.stderr
    cfg = tmp_path / "run.cfg"
    cfg.write_text("factors = 2, 1\niters = 20, 10\nrejection = on\nlog_jacobian = 1\n")
    p = cli("register", tmp_path / "fixed.vol3", tmp_path / "moving.vol3", "--config", cfg,
            "--truth", tmp_path / "u_true.dsp3", "--out-dir", tmp_path / "out")
    assert p.returncode == 0, p.stderr
    summ = dict(kv.split("=", 1) for kv in p.stdout.split())
    assert int(summ["steps"]) == 30 and float(summ["mean_epe"]) >= 0
    first, rows = read_csv(tmp_path / "out" / "trace.csv")
    assert first == "# warplm-csv v1" and len(rows) == 30
    assert list(rows[0]) == ["level", "iter", "loss_raw", "r", "lambda", "eps", "accepted", "retries",
                             "jac_det_min"]
    # the CLI's warp is the API's warp for the same inputs and config
    from paper_2603_19371_b200 import register
    from paper_2603_19371_b200.io import read_dsp3, read_vol3
    res = register(read_vol3(tmp_path / "fixed.vol3"), read_vol3(tmp_path / "moving.vol3"),
                   H._reg_config(H.load_config(str(cfg))))
    assert np.array_equal(np.moveaxis(read_dsp3(tmp_path / "out" / "warp.dsp3"), 0, -1),
                          res.final_warp.astype(np.float32))
    # deterministic
    p2 = cli("register", tmp_path / "fixed.vol3", tmp_path / "moving.vol3", "--config", cfg,
             "--out-dir", tmp_path / "out2")
    assert p2.returncode == 0
    assert (tmp_path / "out" / "trace.csv").read_bytes() == (tmp_path / "out2" / "trace.csv").read_bytes()
    assert (tmp_path / "out" / "warp.dsp3").read_bytes() == (tmp_path / "out2" / "warp.dsp3").read_bytes()


@pytest.mark.gpu
def test_sweep_rows(tmp_path, ctx):
    rows = H.cmd_sweep("lambda0", [1e-4, 0.006, 0.5], repeats=2, dims=(24, 24, 24),
                       csv_path=str(tmp_path / "s.csv"), ctx=ctx)
    assert [(r["value"], r["repeat"]) for r in rows] == [(v, i) for v in (1e-4, 0.006, 0.5) for i in range(2)]
    assert all(np.isfinite(r["mean_epe"]) and r["max_epe"] >= r["mean_epe"] for r in rows)
    first, got = read_csv(tmp_path / "s.csv")
    assert first == "# warplm-csv v1" and list(got[0]) == list(H.SWEEP_COLUMNS) and len(got) == 6


@pytest.mark.gpu
def test_membench_rows(tmp_path):
    rows = H.cmd_membench([32, 64], csv_path=str(tmp_path / "m.csv"))
    for r in rows:
        n = r["n"]
        assert r["state_bytes_lm"] < 1024
        assert r["state_bytes_adam"] == 2 * 3 * n ** 3 * 4  # SPEC.md:447 (6,291,456 at 64)
        assert r["ms_per_step_lm"] > 0 and r["ms_per_step_adam"] > 0
    assert rows[1]["ms_per_step_lm"] <= 1.10 * rows[1]["ms_per_step_adam"]


@pytest.mark.gpu
def test_reject_ablation_rows(tmp_path, ctx):
    rows = H.cmd_reject_ablation(dims=(32, 32, 32), seeds=(0, 1), csv_path=str(tmp_path / "a.csv"), ctx=ctx)
    by = {(r["pair"], r["variant"]): r for r in rows}
    for pair in ("easy-0", "easy-1", "hard"):
        assert by[(pair, "rejection+cap=1.0")]["max_lambda"] <= 1.0
    hard = by[("hard", "rejection+cap=inf")]
    assert hard["max_lambda"] > 1e3 * 0.006 and hard["retries"] > 0
    for pair in ("easy-0", "easy-1"):  # SPEC.md:459 neutrality
        a, b = by[(pair, "no-rejection")]["final_loss"], by[(pair, "rejection+cap=1.0")]["final_loss"]
        assert abs(a - b) < 0.05 * a
    first, got = read_csv(tmp_path / "a.csv")
    assert first == "# warplm-csv v1" and len(got) == 9
