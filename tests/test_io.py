"""VOL3 / DSP3 and the CSV trace (reference io.hpp:15-21, io.cpp:34-109,
SPEC.md:427): the host path runs without a GPU and is checked byte-for-byte
against the unmodified reference io (oracle/_ref) when it is built."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
import paper_2603_19371_b200 as P
from paper_2603_19371_b200 import io as wio

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (reference io.cpp) not built")


def _ref_write(path, data, field):
    L = O.ref_lib()
    err = C.create_string_buffer(256)
    a = np.ascontiguousarray(data, dtype=np.float64)
    shape = a.shape[:3]
    fn = L.ref_write_dsp3 if field else L.ref_write_vol3
    assert fn(os.fsencode(path), a.ctypes.data_as(C.POINTER(C.c_double)), shape[2], shape[1], shape[0],
              err, 256) == 0


def _ref_read(path, field, n):
    L = O.ref_lib()
    err = C.create_string_buffer(256)
    dims = (C.c_int * 3)()
    out = np.empty(n, np.float64)
    rc = L.ref_read(os.fsencode(path), 1 if field else 0, dims, out.ctypes.data_as(C.POINTER(C.c_double)),
                    n, err, 256)
    return rc, tuple(dims), out, err.value.decode()


@needs_ref
def test_vol3_dsp3_bytes_match_reference(tmp_path):
    rng = np.random.default_rng(0)
    vol = rng.normal(size=(5, 6, 7)).astype(np.float32)
    fld = rng.normal(size=(5, 6, 7, 3)).astype(np.float32)  # AoS like DispField3
    for name, data, field in (("a.vol3", vol, False), ("a.dsp3", fld, True)):
        ref, ours = tmp_path / ("ref_" + name), tmp_path / ("ours_" + name)
        _ref_write(ref, data, field)
        if field:
            wio.write_dsp3(ours, np.moveaxis(data, -1, 0))
        else:
            wio.write_vol3(ours, data)
        assert ref.read_bytes() == ours.read_bytes()
        # our reader on the reference's file, the reference's reader on ours
        got = wio.read_dsp3(ref) if field else wio.read_vol3(ref)
        want = np.moveaxis(data, -1, 0) if field else data
        assert np.array_equal(got, want)
        rc, dims, vals, _ = _ref_read(str(ours), field, data.size)
        assert rc == 0 and dims == (7, 6, 5) and np.array_equal(vals, data.reshape(-1).astype(np.float64))


def test_io_errors_match_reference_conditions(tmp_path):
    good = tmp_path / "g.vol3"
    wio.write_vol3(good, np.ones((2, 3, 4), np.float32))
    raw = good.read_bytes()
    cases = {
        "magic": b"XOL3" + raw[4:],
        "header": raw[:10],
        "payload": raw[:-4],
        "dims": raw[:4] + b"\x00\x00\x00\x00" + raw[8:],
        "nonfinite": raw[:16] + np.float32(np.inf).tobytes() + raw[20:],
    }
    for what, blob in cases.items():
        p = tmp_path / f"{what}.vol3"
        p.write_bytes(blob)
        with pytest.raises(wio.IoError):
            wio.read_vol3(p)
    with pytest.raises(wio.IoError):  # a VOL3 is not a DSP3 (magic)
        wio.read_dsp3(good)


def test_trace_csv_schema(tmp_path):
    rows = [dict(level=0, iter=i, loss_raw=0.5 + i, r=0.5 - 0.1 * i, lam=0.006, eps=0.1, accepted=1,
                 retries=0, jac_det_min=float("nan")) for i in range(3)]
    p = tmp_path / "t.csv"
    wio.write_trace_csv(p, rows)
    lines = p.read_text().splitlines()
    assert lines[0] == "# warplm-csv v1"
    assert lines[1] == "level,iter,loss_raw,r,lambda,eps,accepted,retries,jac_det_min"
    vals = lines[3].split(",")
    assert int(vals[1]) == 1 and float(vals[3]) == 0.4 and vals[-1] == "nan"


@pytest.mark.gpu
def test_device_streaming_round_trip(tmp_path, ctx):
    import torch
    rng = np.random.default_rng(1)
    vol = rng.normal(size=(9, 10, 11)).astype(np.float32)
    u = rng.normal(size=(3, 9, 10, 11)).astype(np.float32)
    wio.write_vol3(tmp_path / "v.vol3", vol)
    wio.write_dsp3(tmp_path / "u.dsp3", u)
    dv = torch.empty((9, 10, 11), dtype=torch.float32, device="cuda")
    du = torch.empty((3, 9, 10, 11), dtype=torch.float32, device="cuda")
    wio.read_vol3(tmp_path / "v.vol3", out=dv, ctx=ctx)
    wio.read_dsp3(tmp_path / "u.dsp3", out=du, ctx=ctx)
    assert np.array_equal(dv.cpu().numpy(), vol) and np.array_equal(du.cpu().numpy(), u)
    wio.write_dsp3(tmp_path / "u2.dsp3", du, ctx=ctx)
    wio.write_vol3(tmp_path / "v2.vol3", dv, ctx=ctx)
    assert (tmp_path / "u2.dsp3").read_bytes() == (tmp_path / "u.dsp3").read_bytes()
    assert (tmp_path / "v2.vol3").read_bytes() == (tmp_path / "v.vol3").read_bytes()


@pytest.mark.gpu
def test_register_files(tmp_path, ctx):
    F, M, _ = O.synth_pair((16, 16, 16), 2, num_blobs=6, warp_max=1.5)
    wio.write_vol3(tmp_path / "F.vol3", F)
    wio.write_vol3(tmp_path / "M.vol3", M)
    cfg = P.reg_config(nlevels=2, factors=[2, 1], iters=[5, 5])
    res = wio.register_files(tmp_path / "F.vol3", tmp_path / "M.vol3", tmp_path / "u.dsp3", tmp_path / "t.csv",
                             cfg, ctx=ctx)
    u = wio.read_dsp3(tmp_path / "u.dsp3")
    assert np.array_equal(u, np.moveaxis(res.final_warp, -1, 0).astype(np.float32))
    assert len((tmp_path / "t.csv").read_text().splitlines()) == 2 + len(res.loss_trace)
