"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/wlm.h declares, and the host-only pieces (scalar damping /
rejection state machine, config defaults, state_bytes) behave like the
reference.  No GPU compute is attempted here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "wlm.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(wlm_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    from paper_2603_19371_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares a signature for every exported entry point
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    from paper_2603_19371_b200 import _lib
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_library_built_from_these_sources(monkeypatch):
    """The library carries the hash of the sources it was built from; a stale
    library (sources edited, not rebuilt) is refused at load, not used."""
    from paper_2603_19371_b200 import _lib
    assert C.CDLL(_lib.LIB_PATH).wlm_source_hash  # exported
    lib = _lib.load()
    assert lib.wlm_source_hash().decode() == _lib.source_hash()
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "source_hash", lambda: "0" * 16)
    with pytest.raises(ImportError, match="other sources"):
        _lib.load()


def test_no_gpu_means_loud_failure():
    import paper_2603_19371_b200 as P
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.WlmError):
        P.Context(0)


def test_defaults_match_spec():
    import paper_2603_19371_b200 as P
    c = P.reg_config()
    assert (c.lm.lambda0, c.lm.mu_plus, c.lm.mu_minus) == (0.006, 1.5, 0.975)
    assert (c.lm.tile_size, c.lm.rejection, c.lm.tau, c.lm.lambda_max, c.lm.max_retries) == (1, 0, 1.0, 1.0, 10)
    assert (c.sigma_update, c.sigma_warp) == (1.0, 0.5)
    assert list(c.factors)[:3] == [4, 2, 1] and list(c.iters)[:3] == [100, 75, 50]
    assert (c.target_max_disp, c.step_floor) == (0.4, 1e-12)  # field.hpp:75-78
    assert c.lncc_radius == 2


def test_scalar_state_machine_matches_oracle():
    import oracle as O
    import paper_2603_19371_b200 as P
    rng = np.random.default_rng(0)
    cfgP = P.lm_config()
    cfgO = O.lm_config()
    sP = P.LmState(0.006, 0, 0.0, 0.0)
    sO = O.LmState(0.006, 0, 0.0, 0.0)
    for L in rng.uniform(0.2, 0.4, size=200):
        sP = P.update_damping(sP, L, cfgP)
        sO = O.update_damping(sO, L, cfgO)
        assert (sP.lam, sP.hist_n, sP.L1, sP.L2) == (sO.lam, sO.hist_n, sO.L1, sO.L2)
    for a, b, c_ in rng.uniform(0, 1, size=(200, 3)):
        assert P.rejection_test(a, b, c_, 1.0) == O.rejection_test(a, b, c_, 1.0)


def build_adapter_demo(tmp_path):
    import subprocess
    exe = tmp_path / "adapter_demo"
    lib_dir = os.path.join(ROOT, "paper_2603_19371_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_demo.cpp"), "-L", lib_dir,
                    "-lwarplm_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_adapter_builds(tmp_path):
    """The reference-signature C++ adapter compiles and links against the ABI."""
    assert build_adapter_demo(tmp_path).exists()


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/include/warplm/field.hpp"),
                    reason="reference headers not present")
def test_cpp_adapter_accepts_reference_types(tmp_path):
    """Drop-in: the adapter takes warplm::Volume3 / DispField3 themselves."""
    import subprocess
    src = tmp_path / "drop_in.cpp"
    src.write_text('#include "warplm/field.hpp"\n#include "wlm_warplm.hpp"\n'
                   "double f(const warplm::DispField3& u, const warplm::DispField3& v) {\n"
                   "  warplm::DispField3 w = wlm_warplm::compose_warp(u, v, 0.3);\n"
                   "  warplm::Volume3 s = wlm_warplm::gaussian_smooth(warplm::Volume3(u.dims), 1.0);\n"
                   "  warplm::Volume3 h = wlm_warplm::downsample(s, 2);\n"
                   "  warplm::DispField3 up = wlm_warplm::upsample_warp(w, u.dims, 1.0);\n"
                   "  warplm::DispField3 st = wlm_warplm::lm_step_pointwise(0.5, w, 0.1);\n"
                   "  warplm::Vec3 sf = wlm_warplm::sample_field(up, 0.5, 0.5, 0.5);\n"
                   "  return wlm_warplm::normalize_step(w, warplm::StepScale{}) + s.data[0] + h.data[0]\n"
                   "       + wlm_warplm::sample_trilinear(s, 0.5, 0.5, 0.5) + sf[0] + st.data[0]\n"
                   "       + wlm_warplm::jacobian_det_min(w);\n}\n")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", "/root/reference/proj/include",
                    "-I", os.path.join(ROOT, "include"), str(src)], check=True)


def test_state_bytes():
    import paper_2603_19371_b200 as P
    assert P.state_bytes(P.OPT_ADAM, (64, 64, 64), 4) == 6291456
    assert P.state_bytes(P.OPT_LM, (512, 512, 512), 4) < 1024
    assert P.state_bytes(P.OPT_ADAM, (8, 9, 10), 4) == 2 * 3 * 720 * 4
