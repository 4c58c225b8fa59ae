"""CPU checks of the drop-in boundary: the C-ABI library exists, loads without a GPU, exports every entry point
include/rkfac_b200.h declares, and the product path refuses to run (loudly) without an sm_100 device -- there is no
CPU fallback."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rkfac_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rkfac_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_operator_api():
    fns = declared_functions()
    for f in ("rkfac_ea_update", "rkfac_srevd", "rkfac_rsvd_psd", "rkfac_apply_lowrank_damped_inverse",
              "rkfac_sample_gaussian", "rkfac_plan_step"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    import paper_2206_15397_b200 as rk

    path = rk.LIB_PATH
    if not os.path.exists(path):
        from paper_2206_15397_b200 import build

        build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(rkfac_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_python_bindings_cover_the_header():
    import paper_2206_15397_b200 as rk

    assert sorted(rk.SIGNATURES) == declared_functions()
    lib = rk.load_library()  # loads without a GPU (no CUDA call at load time)
    assert lib.rkfac_status_string(4) == b"DampingNonpositive"


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2206_15397_b200 as rk

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rk.RkfacError):
        rk.context()


def test_status_codes_mirror_reference_exceptions():
    import paper_2206_15397_b200 as rk

    assert rk.DimensionMismatch.status == 1 and rk.RankDeficient.status == 2
    assert rk.NoConvergence.status == 3 and rk.DampingNonpositive.status == 4
    src = open(HEADER).read()
    for name, code in (("RKFAC_DIMENSION_MISMATCH", 1), ("RKFAC_DAMPING_NONPOSITIVE", 4)):
        assert re.search(rf"{name}\s*=\s*{code}", src)


def test_rng_helpers_match_the_oracle(port):
    import paper_2206_15397_b200 as rk

    for s, a, b in ((7, 0, 0), (7, 0, 1), (220615397, 19, 31), (2**63 + 5, 2**40, 3)):
        assert rk.substream_seed(s, a, b) == port.substream(s, a, b)
    assert rk.splitmix64(0) == port.splitmix64(0)


def test_cpp_dropin_compiles_against_reference_headers():
    """include/rkfac_gpu.hpp compiles with the unmodified reference headers (the C++ drop-in boundary)."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers not present on this machine")
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    out = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", ref_inc, "-I", os.path.join(ROOT, "include"),
                          "-I", "/usr/local/cuda/include", src], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-2000:]


def test_c_abi_header_is_plain_c(tmp_path):
    """include/rkfac_b200.h is the FFI boundary: it must compile as C99 (cgo / JNI / ctypes-style hosts), with no
    C++ or torch types in any signature."""
    src = tmp_path / "hdr.c"
    src.write_text('#include "rkfac_b200.h"\nint main(void) { rkfac_factor_desc d; d.dim = 1; return (int)d.dim - 1; }\n')
    out = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only", "-I",
                          os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-2000:]
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    assert "torch" not in text and "std::" not in text and "at::" not in text
